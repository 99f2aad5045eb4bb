// rlfc_field.cu -- fused, tiled, software-pipelined full-field decode (sm_100a).
//
// One CTA owns one TILE: a block row `by` x NB consecutive block columns
// (TW = NB*B pixels wide), for ALL S*T views and all three channels.  The
// reference decodes view by view and re-walks every record once per view
// (kernels.py:219-242 calls decode_chain_core per block per view); here each
// record of the tile is walked once per launch, each present payload is
// BISE-decoded once, and the per-view work is register adds + the colour
// transform.
//
// Setup: the tile's records (three contiguous byte ranges, one per channel;
// container.py:306-323) and its root-plane rows are staged into shared memory
// with 16-byte loads, and one thread per record pre-walks the descriptors of
// levels h-1..k+1 to find where each tree level starts inside its record.
//
// Pipeline, iteration i = 0..T (two CTA barriers per camera row):
//   phase A   walk(i+1)   one thread per record walks the level-0 row i+1 and
//                         any level row that starts at i+1 (one monotone
//                         cursor per level), emitting a work item per present
//                         node into ring E[(i+1)&1]: plain-bit payloads from
//                         the front, trit/quint payloads from the back
//                         (kernels.py:181-215);
//             decode(i)   all threads BISE-decode ring E[i&1], four values per
//                         item with straight-line code per mode, closed-form
//                         bit offsets, digit LUTs in smem, dequantised into the
//                         residual slots of row i (kernels.py:128-159,
//                         202-211); level-0 slots are int32 so the per-view
//                         loop never unpacks;
//   --- barrier ---
//   phase B   blend(i)    (pixel quad, view pair) items: root + levels >= 1 is
//                         a register partial sum shared by the pair, the
//                         level-0 residual is added per view, YCoCg-R inverse
//                         + clamp + pack (colorspace.py:27-56) go to
//                         staging[i&1];
//             store(i-1)  one thread issues ONE 4-D TMA tensor store of the
//                         whole staged row i-1 (all S views x B pixel rows x
//                         TW*3 bytes) straight to HBM, overlapping the blend.
//   --- barrier ---
// Tiles whose records exceed the staging budget, and tiles that saw any stream
// anomaly, run the reference-order per-block walk (walk_chain) so values and
// error precedence are exactly the reference's.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rlfc_common.cuh"
#include "rlfc_field.cuh"

namespace rlfc {

namespace tiled {

#ifdef RLFC_PHASE_TIMING
__device__ long long g_phase[4096 * 8 * 8];
#endif

constexpr int MAXH = 8;        // tree levels handled by the tiled kernel
constexpr int MAXS = 64;       // camera columns handled by the tiled kernel

struct Params {
    rlfc_field f;
    int stop_level;
    const int32_t* slots;
    int by_lo;
    uint8_t* rgb;
    int64_t img_stride, row_stride;
    uint64_t* status;
    int tiles_x;
    int off_nbt, off_cur, off_err, off_cnt, off_mask, off_ent, off_root, off_rgb, off_list, off_res0, off_resl,
        off_stage, off_bytes, off_mbar;
    int bytes_cap, ent_cap, seg_cap, off_priv;
    int slot_base[MAXH];       // level l >= 1: first slot of its row in resl
    int store_mode;            // 2: one 4-D TMA tensor store per row, 1: per-row
                               // cp.async.bulk, 0: byte stores (unaligned rows)
    int roots_all;             // 1: every root of the tile is staged at setup
    int roots_vec;             // 1: root rows are 16-byte aligned in HBM
    int no_prefill;            // tuning build only (RLFC_TUNING): every view dirty
    int specialized;           // 1: dedicated walker warps (named-barrier handoff)
};

// One decode job: payload byte offset in the staged tile (16 bits), descriptor
// (5), channel (2), block (3), residual slot (6; slot < S is the level-0 row,
// else a level row at slot - S).
using Entry = uint32_t;
__device__ __forceinline__ Entry make_entry(uint32_t off, int d, int c, int b, int slot) {
    return off | (uint32_t)d << 16 | (uint32_t)c << 21 | (uint32_t)b << 23 | (uint32_t)slot << 26;
}

// 32 bits at bit position `bitpos` of the 16-byte aligned staging buffer.
__device__ __forceinline__ uint32_t sbits(const uint32_t* w, uint32_t bitpos) {
    const uint32_t i = bitpos >> 5;
    return __funnelshift_r(w[i], w[i + 1], bitpos & 31u);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Clamp four int32 to [0, 255] and pack them little-endian into one word
// (cvt.pack.sat: saturating convert + pack, two instructions).
__device__ __forceinline__ uint32_t pack4_sat(int32_t b0, int32_t b1, int32_t b2, int32_t b3) {
    uint32_t hi, d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(hi) : "r"(b3), "r"(b2), "r"(0));
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(b1), "r"(b0), "r"(hi));
    return d;
}

// kernels.py:202-211 dequantisation in 32-bit wrap arithmetic: identical to
// the reference's int64 result truncated into its int32 accumulator.
__device__ __forceinline__ int32_t deq(uint32_t z, int shift) {
    if (shift >= 32) return dequant(z, shift);
    const uint32_t mag = (((z + 1u) >> 1) << shift) + ((1u << shift) >> 1);
    const uint32_t v = (z & 1u) ? 0u - mag : mag;
    return z ? (int32_t)v : 0;
}

template <int B, int TW>
struct Cfg {
    static constexpr int NB = TW / B;           // blocks per tile
    static constexpr int NREC = 3 * NB;         // records per tile
    static constexpr int BSQ = B * B;
    static constexpr int QPB = BSQ / 4;         // value quads per block
    static constexpr int QPR = TW / 4;          // pixel quads per tile row
    static constexpr int QUADS = QPR * B;       // pixel quads per tile
    static constexpr int MAX_THREADS = 256;
    static_assert(NREC <= 32, "walkers live in one warp");
};

template <typename T>
__device__ __forceinline__ void load4(const T* p, int32_t* v);
template <>
__device__ __forceinline__ void load4<int16_t>(const int16_t* p, int32_t* v) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
    v[0] = (int32_t)(int16_t)(w.x & 0xFFFFu);
    v[1] = (int32_t)w.x >> 16;
    v[2] = (int32_t)(int16_t)(w.y & 0xFFFFu);
    v[3] = (int32_t)w.y >> 16;
}
template <>
__device__ __forceinline__ void load4<int32_t>(const int32_t* p, int32_t* v) {
    const int4 w = *reinterpret_cast<const int4*>(p);
    v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
}
template <typename T>
__device__ __forceinline__ void store4(T* p, const int32_t* v);
template <>
__device__ __forceinline__ void store4<int16_t>(int16_t* p, const int32_t* v) {
    uint2 w;
    w.x = ((uint32_t)v[0] & 0xFFFFu) | ((uint32_t)v[1] << 16);
    w.y = ((uint32_t)v[2] & 0xFFFFu) | ((uint32_t)v[3] << 16);
    *reinterpret_cast<uint2*>(p) = w;
}
template <>
__device__ __forceinline__ void store4<int32_t>(int32_t* p, const int32_t* v) {
    *reinterpret_cast<int4*>(p) = make_int4(v[0], v[1], v[2], v[3]);
}

// Reference-order fallback for one tile: one thread per (view, block), three
// chains walked from global memory exactly as kernels.py:162-216; writes the
// values and reports the exact failure key.
template <int B>
__device__ __noinline__ void tile_fallback(const Params& P, int by, int bx0, int nb, const DigitLut& lut,
                                           const NodeBytes& nb_tab) {
    const rlfc_field& f = P.f;
    const int nimg = f.s_count * f.t_count;
    for (int job = threadIdx.x; job < nimg * nb; job += blockDim.x) {
        const int img = job / nb, bx = bx0 + job % nb;
        const int slot = P.slots ? P.slots[img] : img;
        if (slot < 0) continue;
        const int s = img / f.t_count, t = img % f.t_count;
        int32_t acc[3][B * B];
        bool bad = false;
        for (int c = 0; c < 3 && !bad; ++c) {
            for (int yy = 0; yy < B; ++yy)
                for (int xx = 0; xx < B; ++xx) acc[c][yy * B + xx] = root_sample(f, s, t, c, by * B + yy, bx * B + xx);
            const uint64_t off = f.offsets[c][by * f.wb + bx];
            int st = walk_chain<B * B>(f, f.srv[c] + off, s, t, P.stop_level, acc[c], lut, nb_tab,
                                       srv_avail(f, c, off));
            if (st == WALK_OOB) st = 2;
            if (st) {
                report(P.status, (((uint64_t)img * 3 + c) * f.hb + by) * f.wb + bx, st);
                bad = true;
            }
        }
        if (bad) continue;
        uint8_t* o = P.rgb + (int64_t)slot * P.img_stride;
        for (int yy = 0; yy < B; ++yy) {
            const int y = by * B + yy;
            if (y >= f.height) break;
            uint8_t* orow = o + (int64_t)(y - P.by_lo * B) * P.row_stride;
            for (int xx = 0; xx < B; ++xx) {
                const int x = bx * B + xx;
                if (x >= f.width) break;
                uint32_t r, g, b;
                const int j = yy * B + xx;
                ycocg_to_rgb8(acc[0][j], acc[1][j], acc[2][j], r, g, b);
                orow[3 * x] = (uint8_t)r;
                orow[3 * x + 1] = (uint8_t)g;
                orow[3 * x + 2] = (uint8_t)b;
            }
        }
    }
}

template <int B, int TW, typename VT, typename RT>
__global__ void __launch_bounds__(Cfg<B, TW>::MAX_THREADS)
    k_decode_field_tiled(const __grid_constant__ Params P, const __grid_constant__ CUtensorMap out_map) {
    using C = Cfg<B, TW>;
    extern __shared__ __align__(128) uint8_t smem[];
    const rlfc_field& f = P.f;
    const int tid = threadIdx.x;
    const int THREADS = blockDim.x;
    // specialized launch: warps 0..NCONS/32-1 consume (decode, classify,
    // blend, store); the last two warps only walk, running ahead of them
    const int NCONS = P.specialized ? THREADS - 64 : THREADS;
    const int by = P.by_lo + blockIdx.x / P.tiles_x;
    const int bx0 = (blockIdx.x % P.tiles_x) * C::NB;
    const int nb = min(C::NB, f.wb - bx0);
    const int k = P.stop_level, h = f.tree_height;
    const int S = f.s_count, T = f.t_count;
    const int lmin = k > 0 ? k : 1;              // levels >= lmin are held as full rows
    const int plane = 3 * B * TW;                // values per slot / root ([3][B][TW])

    DigitLut& lut = *reinterpret_cast<DigitLut*>(smem);
    NodeBytes& nbt = *reinterpret_cast<NodeBytes*>(smem + P.off_nbt);
    uint32_t* cur = reinterpret_cast<uint32_t*>(smem + P.off_cur);   // [NREC][MAXH]
    int32_t* err = reinterpret_cast<int32_t*>(smem + P.off_err);     // [NREC]
    // cnt[0..1]: plain-bit entries of ring 0/1 (front), cnt[2..3]: trit/quint
    // entries (back), cnt[4]: anomaly flag, cnt[5]/[6]: dirty / clean items
    int32_t* cnt = reinterpret_cast<int32_t*>(smem + P.off_cnt);
    uint32_t* mask = reinterpret_cast<uint32_t*>(smem + P.off_mask); // [2 ring][MAXH][NREC][2]
    Entry* ent = reinterpret_cast<Entry*>(smem + P.off_ent);         // [2 ring][ent_cap]
    RT* roots = reinterpret_cast<RT*>(smem + P.off_root);            // [root][3][B][TW]
    uint32_t* root_rgb = reinterpret_cast<uint32_t*>(smem + P.off_rgb); // [root][B][TW*3/4] packed RGB8
    uint2* lists = reinterpret_cast<uint2*>(smem + P.off_list);      // [S*NB]: dirty from 0, clean from the end
    VT* res0 = reinterpret_cast<VT*>(smem + P.off_res0);             // [s][3][B][TW]
    VT* resl = reinterpret_cast<VT*>(smem + P.off_resl);             // [slot][3][B][TW]
    uint8_t* stage = smem + P.off_stage;                             // [S][B][TW*3]
    uint8_t* bytes = smem + P.off_bytes;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(bytes);

    // ---- tables -------------------------------------------------------------
    {
        uint16_t* l16 = reinterpret_cast<uint16_t*>(smem);
        for (int i = tid; i < 243 + 125; i += THREADS) {
            int p, v = 0;
            if (i < 243) {
                p = i;
                for (int d = 0; d < 5; ++d) { v |= (p % 3) << (2 * d); p /= 3; }
            } else {
                p = i - 243;
                for (int d = 0; d < 3; ++d) { v |= (p % 5) << (3 * d); p /= 5; }
            }
            l16[i] = (uint16_t)v;
        }
        if (tid < 32) nbt.v[tid] = tid < NUM_DESC ? (uint16_t)(1 + payload_bytes(tid, B * B)) : (uint16_t)0;
        if (tid < 8) cnt[tid] = 0;
    }
    // ---- the tile's record bytes --------------------------------------------
    uint64_t abeg[3], aend[3], tend[3];
    uint32_t sbase[3];
    uint64_t total = 0;
    bool range_ok = true;
    const bool need_srv = k < h;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t blk0 = (int64_t)by * f.wb + bx0;
        const uint64_t beg = f.offsets[c][blk0];
        const uint64_t end = (blk0 + nb < (int64_t)f.wb * f.hb) ? f.offsets[c][blk0 + nb] : f.srv_len[c];
        range_ok &= beg <= end && end <= f.srv_len[c];
        tend[c] = end;
        abeg[c] = beg & ~uint64_t(15);
        aend[c] = (end + 15) & ~uint64_t(15);
        sbase[c] = (uint32_t)total;
        total += need_srv && range_ok ? aend[c] - abeg[c] : 0u;
    }
    __syncthreads();
    // does not fit, or the offsets leave the section: reference-order walk
    if ((need_srv && !range_ok) || total + 16 > (uint64_t)P.bytes_cap) {
        tile_fallback<B>(P, by, bx0, nb, lut, nbt);
        return;
    }
    if (need_srv) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const uint4* src = reinterpret_cast<const uint4*>(f.srv[c] + abeg[c]);
            uint4* dst = reinterpret_cast<uint4*>(bytes + sbase[c]);
            const uint32_t n16 = (uint32_t)((aend[c] - abeg[c]) >> 4);
            for (uint32_t i = tid; i < n16; i += THREADS) dst[i] = __ldg(src + i);
        }
    }
    // root rows of the tile: [root (rx*rsy + ry)][c][row][TW]; all of them at
    // setup when they fit, else one root row (ry) at a time in decode()
    const bool full_tile = (bx0 + C::NB) * B <= f.wp;
    auto load_roots = [&](int ry0, int nry, RT* dst) {
        const int64_t pl = (int64_t)f.hp * f.wp;
        const int segs = nry * f.rsx * 3 * B;            // (ry, rx, c, row) segments of TW values
        if (P.roots_vec && full_tile) {
            constexpr int V = TW * (int)sizeof(RT) / 16;   // uint4 per segment
            for (int i = tid; i < segs * V; i += THREADS) {
                const int v = i % V, sg = i / V;
                const int rr = sg % B, c = (sg / B) % 3, rx = (sg / (3 * B)) % f.rsx, ry = ry0 + sg / (3 * B * f.rsx);
                const RT* src = reinterpret_cast<const RT*>(f.roots) +
                                (((int64_t)rx * f.rsy + ry) * 3 + c) * pl + (int64_t)(by * B + rr) * f.wp + bx0 * B;
                const int droot = P.roots_all ? rx * f.rsy + ry : rx;
                reinterpret_cast<uint4*>(dst + ((droot * 3 + c) * B + rr) * TW)[v] =
                    __ldg(reinterpret_cast<const uint4*>(src) + v);
            }
        } else {
            for (int i = tid; i < segs * TW; i += THREADS) {
                const int x = i % TW, sg = i / TW;
                const int rr = sg % B, c = (sg / B) % 3, rx = (sg / (3 * B)) % f.rsx, ry = ry0 + sg / (3 * B * f.rsx);
                const int gx = bx0 * B + x;
                RT v = 0;
                if (gx < f.wp)
                    v = reinterpret_cast<const RT*>(f.roots)[(((int64_t)rx * f.rsy + ry) * 3 + c) * pl +
                                                             (int64_t)(by * B + rr) * f.wp + gx];
                const int droot = P.roots_all ? rx * f.rsy + ry : rx;
                dst[((droot * 3 + c) * B + rr) * TW + x] = v;
            }
        }
    };
    if (P.roots_all) load_roots(0, f.rsy, roots);
    // walkers: one thread per (channel, block) record.  The last warp walks
    // the lowest level's row (level 0, or the stop level), the warp before it
    // walks the level rows above; the pre-walk is done by the last warp.
    const int wid = tid - (THREADS - 32);                    // lane in the last warp
    const int wid2 = tid - (THREADS - 64);                   // lane in the warp before
    const bool walker = wid >= 0 && wid < C::NREC && (wid % C::NB) < nb && need_srv;
    const bool walker2 = wid2 >= 0 && wid2 < C::NREC && (wid2 % C::NB) < nb && need_srv;
    const int wrec = walker ? wid : (walker2 ? wid2 : 0);
    const int wc = wrec / C::NB, wblk = wrec % C::NB;
    uint32_t my_beg = 0, my_len = 0;
    if (walker || walker2) {
        const int64_t blk = (int64_t)by * f.wb + bx0 + wblk;
        const uint64_t rb = f.offsets[wc][blk];
        const uint64_t re = (blk + 1 < (int64_t)f.wb * f.hb) ? f.offsets[wc][blk + 1] : f.srv_len[wc];
        // a record outside the tile's staged range (non-monotone offsets)
        // gets length 0: the pre-walk flags it and the tile falls back
        if (rb >= abeg[wc] && rb <= re && re <= tend[wc]) {
            my_beg = sbase[wc] + (uint32_t)(rb - abeg[wc]);
            my_len = (uint32_t)(re - rb);
        }
    }
    if (tid < C::NREC) err[tid] = 0;
    __syncthreads();

    // ---- pre-walk: start of each level inside each record -------------------
    uint32_t* mycur = cur + wrec * MAXH;
    if (walker) {
        const uint8_t* rec = bytes + my_beg;
        const uint32_t rbit = my_beg << 3;
        uint32_t cu = (uint32_t)f.bitmap_bytes;
        bool bad = cu > my_len;
        mycur[h - 1] = cu;
        for (int l = h - 1; l > k && !bad; --l) {
            const int n0 = f.level_base[l], n1 = n0 + f.level_sx[l] * f.level_sy[l];
            for (int w = n0; w < n1 && !bad; w += 32) {
                uint32_t bits = sbits(words, rbit + (uint32_t)w);
                if (n1 - w < 32) bits &= (1u << (n1 - w)) - 1u;
                while (bits) {
                    bits &= bits - 1u;
                    const int d = cu < my_len ? rec[cu] : NUM_DESC;
                    if (d >= NUM_DESC || cu + nbt.v[d] > my_len) { bad = true; break; }
                    cu += nbt.v[d];
                }
            }
            mycur[l - 1] = cu;
        }
        if (bad) { err[wid] = 1; cnt[4] = 1; }
    }

    // walk(t): the level rows that start at t (warp before last) and the
    // lowest level's row t (last warp) -> ring t&1.  Each walker lane keeps
    // its entries in a private segment; a warp scan then places them in the
    // ring (plain-bit payloads from the front, trit/quint from the back) with
    // one atomic per warp.  Level-l masks live in ring ((t >> l) & 1): a row's
    // mask stays valid for all 2^l camera rows that use it.
    // Ring of work items for parity p = t & 1: one segment per (walker group,
    // record) -- plain-bit entries grow from the front of a segment,
    // trit/quint entries from its back -- and, per group and kind, the
    // exclusive prefix of the records' entry counts ([NREC] = group total).
    const int seg_cap = P.seg_cap;
    auto seg_of = [&](int p, int g, int r) -> Entry* {
        return ent + ((size_t)(p * 2 + g) * C::NREC + r) * seg_cap;
    };
    auto pre_of = [&](int p, int g, int kind) -> int32_t* {
        return reinterpret_cast<int32_t*>(smem + P.off_priv) + ((p * 2 + g) * 2 + kind) * 32;
    };
    auto walk = [&](int t) {
        if (tid < THREADS - 64) return;                  // only the two walker warps
        const bool low = walker, up = walker2;
        const int g = (tid >= THREADS - 32) ? 0 : 1;     // 0: lowest level row, 1: level rows
        const bool active = (low || up) && !err[wrec];
        const uint8_t* rec = bytes + my_beg;
        const uint32_t rbit = my_beg << 3;
        Entry* seg = seg_of(t & 1, g, wrec);
        int nbits = 0, ntq = 0;
        bool bad = false;
        const int lo_l = low ? k : k + 1, hi_l = low ? k : h - 1;
        for (int l = hi_l; active && l >= lo_l && !bad; --l) {
            if (!low && (t & ((1 << l) - 1)) != 0) continue;   // level row not due
            const bool row_level = l >= lmin;
            if (low && row_level && (t & ((1 << l) - 1)) != 0) continue;   // k >= 1: lowest row level
            const int sx = f.level_sx[l];
            const int n0 = f.level_base[l] + (t >> l) * sx;
            const int sb = row_level ? S + P.slot_base[l] : 0;
            uint32_t cu = mycur[l];
            uint32_t mw0 = 0u, mw1 = 0u;
            for (int w = 0; w < sx && !bad; w += 32) {
                uint32_t bits = sbits(words, rbit + (uint32_t)(n0 + w));
                if (sx - w < 32) bits &= (1u << (sx - w)) - 1u;
                if (w == 0) mw0 = bits;
                else mw1 = bits;
                while (bits) {
                    const int x = w + __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const int d = cu < my_len ? rec[cu] : NUM_DESC;
                    if (d >= NUM_DESC || cu + nbt.v[d] > my_len) { bad = true; break; }
                    const Entry en = make_entry(my_beg + cu + 1, d, wc, wblk, sb + x);
                    if (desc_mode(d) == MODE_BITS) seg[nbits++] = en;
                    else seg[seg_cap - 1 - (ntq++)] = en;
                    cu += nbt.v[d];
                }
            }
            mycur[l] = cu;
            uint32_t* M = mask + (((t >> l) & 1) * MAXH + l) * C::NREC * 2 + wrec * 2;
            M[0] = mw0;
            M[1] = mw1;
        }
        if (bad) { err[wrec] = 1; cnt[4] = 1; }
        // exclusive prefix of the per-record counts (idle lanes count 0)
        const int lane = tid & 31;
        int ib = (low || up) ? nbits : 0, iq = (low || up) ? ntq : 0;
        const int cb = ib, cq = iq;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yb = __shfl_up_sync(0xffffffffu, ib, o), yq = __shfl_up_sync(0xffffffffu, iq, o);
            if (lane >= o) { ib += yb; iq += yq; }
        }
        int32_t* pb = pre_of(t & 1, g, 0);
        int32_t* pq = pre_of(t & 1, g, 1);
        if (lane < C::NREC) {
            pb[lane] = ib - cb;
            pq[lane] = iq - cq;
        }
        if (lane == 31) {
            pb[C::NREC] = ib;
            pq[C::NREC] = iq;
        }
    };

    // decode(t): ring t&1 -> residual slots (+ the root row when it starts).
    // One item = 4 consecutive values of one payload (one pixel-row quad of
    // its block).
    const int shift = f.quant_shift;
    auto put = [&](Entry en, int j, const int32_t* v) {
        const int c = (en >> 21) & 3, b = (en >> 23) & 7, slot = en >> 26;
        const int row = (4 * j) / B, col = (4 * j) % B;
        const int o = (c * B + row) * TW + b * B + col;
        if (slot < S) store4<VT>(res0 + slot * plane + o, v);
        else store4<VT>(resl + (slot - S) * plane + o, v);
    };
    // find the record owning entry e of (group g, kind) at parity p: the
    // last r with prefix[r] <= e
    auto owner = [&](const int32_t* pre, int e) -> int {
        int r = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
            if (r + step < C::NREC && pre[r + step] <= e) r += step;
        return r;
    };
    auto decode = [&](int t) {
        const int p = t & 1;
        const int32_t *pb0 = pre_of(p, 0, 0), *pb1 = pre_of(p, 1, 0);
        const int32_t *pq0 = pre_of(p, 0, 1), *pq1 = pre_of(p, 1, 1);
        const int nb0 = pb0[C::NREC], nf = nb0 + pb1[C::NREC];
        const int nq0 = pq0[C::NREC], nbk = nq0 + pq1[C::NREC];
        const int items_f = nf * C::QPB, items = items_f + nbk * C::QPB;
        for (int it = tid; it < items; it += NCONS) {
            int32_t v[4];
            if (it < items_f) {
                // plain b-bit fields: the quad's 4b <= 44 bits in one 64-bit window
                const int e = it / C::QPB, j = it - e * C::QPB;
                const int g = e < nb0 ? 0 : 1, eg = e - (g ? nb0 : 0);
                const int32_t* pre = g ? pb1 : pb0;
                const int r = owner(pre, eg);
                const Entry en = seg_of(p, g, r)[eg - pre[r]];
                const int b = desc_bits((en >> 16) & 31);
                const uint32_t p0 = ((en & 0xFFFFu) << 3) + (uint32_t)(4 * j * b);
                const uint64_t win = (uint64_t)sbits(words, p0) | ((uint64_t)sbits(words, p0 + 32) << 32);
                const uint32_t lm = (1u << b) - 1u;
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = deq((uint32_t)(win >> (i * b)) & lm, shift);
                put(en, j, v);
            } else {
                const int it2 = it - items_f;
                const int e = it2 / C::QPB, j = it2 - e * C::QPB;
                const int g = e < nq0 ? 0 : 1, eg = e - (g ? nq0 : 0);
                const int32_t* pre = g ? pq1 : pq0;
                const int r = owner(pre, eg);
                const Entry en = seg_of(p, g, r)[seg_cap - 1 - (eg - pre[r])];
                const int d = (en >> 16) & 31;
                const bool trit = desc_mode(d) == MODE_TRIT;
                const int b = desc_bits(d);
                const uint32_t G = trit ? 5u : 3u, PBITS = trit ? 8u : 7u, DB = trit ? 2u : 3u;
                const uint32_t PMAX = trit ? 242u : 124u, DMASK = trit ? 3u : 7u;
                const uint32_t MAGIC = trit ? 13108u : 21846u;            // kk/G, kk < 256
                const uint16_t* L = trit ? lut.trit : lut.quint;
                const uint32_t gbits = PBITS + G * (uint32_t)b;
                const uint32_t base = (en & 0xFFFFu) << 3, lm = (1u << b) - 1u;
                const uint32_t k0 = 4u * (uint32_t)j;
                const uint32_t g0 = (k0 * MAGIC) >> 16, g1 = ((k0 + 3u) * MAGIC) >> 16;
                const uint32_t pk0 = sbits(words, base + g0 * gbits) & ((1u << PBITS) - 1u);
                const uint32_t pk1 = sbits(words, base + g1 * gbits) & ((1u << PBITS) - 1u);
                if (pk0 > PMAX || pk1 > PMAX) {           // kernels.py:147-150
                    err[((en >> 21) & 3) * C::NB + ((en >> 23) & 7)] = 1;
                    cnt[4] = 1;
                }
                const uint32_t dg0 = L[pk0 <= PMAX ? pk0 : 0u], dg1 = L[pk1 <= PMAX ? pk1 : 0u];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t kk = k0 + (uint32_t)i;
                    const uint32_t gg = (kk * MAGIC) >> 16, ii = kk - gg * G;
                    const uint32_t digit = ((gg == g0 ? dg0 : dg1) >> (DB * ii)) & DMASK;
                    const uint32_t low = sbits(words, base + gg * gbits + PBITS + ii * (uint32_t)b) & lm;
                    v[i] = deq((digit << b) | low, shift);
                }
                put(en, j, v);
            }
        }
        if (!P.roots_all && (t & ((1 << h) - 1)) == 0) load_roots(t >> h, 1, roots);
    };

    // Root colours: RGB(root) of every root of the tile, computed once at setup
    // (roots_all).  Most (view, block) pairs carry no residual at any level:
    // their pixels are exactly RGB(root), so each view's staging rows start as
    // a copy of RGB(root) (prefill) and the threads overwrite only the DIRTY
    // (view, block) pairs.
    const bool use_rgb = P.roots_all != 0 && !P.no_prefill;
    if (use_rgb) {
        const int nroot = f.rsx * f.rsy;
        for (int it = tid; it < nroot * B * C::QPR; it += THREADS) {
            const int xq = it % C::QPR, rr = (it / C::QPR) % B, ri = it / (C::QPR * B);
            const RT* rp = roots + (size_t)ri * plane + rr * TW + xq * 4;
            int32_t v[3][4];
#pragma unroll
            for (int c = 0; c < 3; ++c) load4<RT>(rp + c * B * TW, v[c]);
            int32_t o[12];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int32_t tt = v[0][i] - (v[2][i] >> 1);
                const int32_t bb = tt - (v[1][i] >> 1);
                o[3 * i] = bb + v[1][i];
                o[3 * i + 1] = v[2][i] + tt;
                o[3 * i + 2] = bb;
            }
            uint32_t* d = root_rgb + (ri * B + rr) * (TW * 3 / 4) + xq * 3;
            d[0] = pack4_sat(o[0], o[1], o[2], o[3]);
            d[1] = pack4_sat(o[4], o[5], o[6], o[7]);
            d[2] = pack4_sat(o[8], o[9], o[10], o[11]);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

    // views of row t the caller wants (64-bit mask over s), warp-wide
    const uint64_t all_views = S >= 64 ? ~0ull : ((1ull << S) - 1ull);
    auto want_mask = [&](int t) -> uint64_t {
        if (!P.slots) return all_views;
        const int lane = tid & 31;
        const bool w0 = lane < S && (!P.slots || P.slots[lane * T + t] >= 0);
        const bool w1 = lane + 32 < S && (!P.slots || P.slots[(lane + 32) * T + t] >= 0);
        return (uint64_t)__ballot_sync(0xffffffffu, w0) | (uint64_t)__ballot_sync(0xffffffffu, w1) << 32;
    };

    // prefill(t): staging[t&1][s] <- RGB(root(s, t)) for every view, 16-byte
    // cooperative copies (dirty blocks are overwritten by blend(t))
    auto prefill = [&](int t) {
        if (!use_rgb) return;
        uint4* stg = reinterpret_cast<uint4*>(stage);
        const int ry = t >> h;
        constexpr int V = B * TW * 3 / 16;               // uint4 per view
        for (int it = tid; it < S * V; it += NCONS) {
            const int sv = it / V, v = it - sv * V;
            stg[it] = reinterpret_cast<const uint4*>(root_rgb + ((sv >> h) * f.rsy + ry) * (V * 4))[v];
        }
    };

    // classify(t), two steps.  (1) lanes 0..nb-1 of warp 0 build, per block,
    // the 64-bit mask of views whose chain carries any residual in any
    // channel (level-l row bits spread over their 2^l views); (2) after the
    // phase barrier every thread takes (view, block) items, keeps the dirty
    // ones and appends them -- with their presence bits (bit 3l+c: level l,
    // channel c) -- by warp-aggregated atomics (order is irrelevant).
    uint64_t* dmask = reinterpret_cast<uint64_t*>(lists + S * C::NB);   // [NB]
    int32_t* dpre = reinterpret_cast<int32_t*>(dmask + C::NB);          // [NB] exclusive prefix
    auto classify_masks = [&](int t, uint64_t want) {
        if (tid >= 32) return;
        const int b = tid;
        uint64_t dirty = 0;
        if (b < nb) {
            if (!use_rgb) {
                dirty = want;
            } else {
                for (int l = h - 1; l >= k; --l) {
                    const uint32_t* M = mask + (((t >> l) & 1) * MAXH + l) * C::NREC * 2;
                    uint64_t ml = 0;
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        ml |= (uint64_t)M[(c * C::NB + b) * 2] | (uint64_t)M[(c * C::NB + b) * 2 + 1] << 32;
                    if (l == 0) {
                        dirty |= ml;
                    } else {
                        const int span = 1 << l;
                        const uint64_t run = span >= 64 ? ~0ull : ((1ull << span) - 1ull);
                        while (ml) {
                            const int x = __ffsll((long long)ml) - 1;
                            ml &= ml - 1;
                            const int s0 = x << l;
                            if (s0 < 64) dirty |= run << s0;
                        }
                    }
                }
                dirty &= want;
            }
        }
        const int n = __popcll(dirty);
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += y;
        }
        if (b < C::NB) {
            dmask[b] = dirty;
            dpre[b] = incl - n;
        }
        if (tid == 31) cnt[5] = incl;
    };
    // classify_items(t): thread i takes dirty item i: its block from the
    // prefix, its view as the k-th set bit of the block's mask, then its
    // presence bits (bit 3l+c: level l, channel c)
    auto classify_items = [&](int t) {
        const int total = cnt[5];
        for (int i = tid; i < total; i += NCONS) {
            int b = 0;
#pragma unroll
            for (int j = 1; j < C::NB; ++j) b += (dpre[j] <= i) ? 1 : 0;
            const int kth = i - dpre[b];
            uint64_t m = dmask[b];
            for (int j = 0; j < kth; ++j) m &= m - 1;        // drop the kth lowest views
            const int sv = __ffsll((long long)m) - 1;
            uint32_t pres = 0;
            for (int l = h - 1; l >= k; --l) {
                const int x = sv >> l;
                const uint32_t* M = mask + (((t >> l) & 1) * MAXH + l) * C::NREC * 2;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    pres |= ((M[(c * C::NB + b) * 2 + (x >> 5)] >> (x & 31)) & 1u) << (3 * l + c);
            }
            lists[i] = make_uint2((uint32_t)sv | (uint32_t)b << 8, pres);
        }
    };

    // blend(t), phase B: tasks = (dirty item, pixel quad of its block): root +
    // present residuals, colorspace.py:27-36 inverse lift, clamp, pack.
    constexpr int QB = B / 4;                           // quads per block row
    auto blend = [&](int t) {
        const int tasks = cnt[5] * C::QPB;
        __syncwarp();
        uint8_t* stg = stage;
        const RT* rrow = roots + (P.roots_all ? (t >> h) : 0) * plane;
        for (int it = tid; it < tasks; it += NCONS) {
            const int li = it / C::QPB, j = it - li * C::QPB;
            const uint2 item = lists[li];
            const int sv = item.x & 255, bv = (item.x >> 8) & 255;
            const int row = j / QB, colq = (j % QB) * 4;
            const int px = bv * B + colq;                   // pixel column in the tile
            uint32_t* sp = reinterpret_cast<uint32_t*>(stg + (sv * B + row) * (TW * 3) + px * 3);
            const int rx = sv >> h;
            const uint32_t pres = item.y;
            const int poff = row * TW + px;
            const int root_idx = P.roots_all ? rx * f.rsy : rx;
            int32_t v[3][4];
#pragma unroll
            for (int c = 0; c < 3; ++c) load4<RT>(rrow + (root_idx * 3 + c) * B * TW + poff, v[c]);
            uint32_t lv = (pres >> 3) & ~0u;            // levels >= 1
            while (lv) {
                const int bit = __ffs(lv) - 1;
                const int l = 1 + bit / 3;
                const uint32_t pl = (pres >> (3 * l)) & 7u;
                lv &= ~(7u << (3 * (l - 1)));
                const VT* rp = resl + (P.slot_base[l] + (sv >> l)) * plane + poff;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    int32_t r[4] = {0, 0, 0, 0};
                    if ((pl >> c) & 1u) load4<VT>(rp + c * B * TW, r);
#pragma unroll
                    for (int i = 0; i < 4; ++i) v[c][i] += r[i];
                }
            }
            if (pres & 7u) {
                const VT* rp = res0 + sv * plane + poff;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    int32_t r[4] = {0, 0, 0, 0};
                    if ((pres >> c) & 1u) load4<VT>(rp + c * B * TW, r);
#pragma unroll
                    for (int i = 0; i < 4; ++i) v[c][i] += r[i];
                }
            }
            int32_t o[12];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int32_t tt = v[0][i] - (v[2][i] >> 1);
                const int32_t bb = tt - (v[1][i] >> 1);
                o[3 * i] = bb + v[1][i];
                o[3 * i + 1] = v[2][i] + tt;
                o[3 * i + 2] = bb;
            }
            sp[0] = pack4_sat(o[0], o[1], o[2], o[3]);
            sp[1] = pack4_sat(o[4], o[5], o[6], o[7]);
            sp[2] = pack4_sat(o[8], o[9], o[10], o[11]);
        }
    };

    // store(t): staging[t&1] -> HBM (true-dims crop)
    const int row_bytes = min(TW, f.width - bx0 * B) * 3;
    const int mode = P.store_mode == 1 && row_bytes != TW * 3 ? 0 : P.store_mode;
    bool issued = false;
    auto store = [&](int t) {
        const uint8_t* stg = stage;
        if (mode == 2) {
            // one TMA tensor store: box (TW*3 bytes, B rows, 1 camera row, S
            // columns) at (x0, y0, t, 0); TMA clips the right / bottom edges
            if (tid == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                        &out_map),
                    "r"(bx0 * B * 3), "r"((by - P.by_lo) * B), "r"(t), "r"(0), "r"(smem_addr(stg))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                issued = true;
            }
        } else if (mode == 1) {
            for (int it = tid; it < S * B; it += NCONS) {
                const int s = it / B, rr = it % B;
                const int y = by * B + rr;
                const int img = s * T + t;
                const int slot = P.slots ? P.slots[img] : img;
                if (slot < 0 || y >= f.height) continue;
                uint8_t* orow = P.rgb + (int64_t)slot * P.img_stride + (int64_t)(y - P.by_lo * B) * P.row_stride +
                                (int64_t)bx0 * B * 3;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(orow),
                             "r"(smem_addr(stg + (s * B + rr) * (TW * 3))), "n"(TW * 3)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                issued = true;
            }
        } else {
            for (int it = tid; it < S * B * (TW * 3); it += NCONS) {
                const int bcol = it % (TW * 3), rr = (it / (TW * 3)) % B, s = it / (TW * 3 * B);
                const int y = by * B + rr;
                if (bcol >= row_bytes || y >= f.height) continue;
                const int img = s * T + t;
                const int slot = P.slots ? P.slots[img] : img;
                if (slot < 0) continue;
                P.rgb[(int64_t)slot * P.img_stride + (int64_t)(y - P.by_lo * B) * P.row_stride +
                      (int64_t)bx0 * B * 3 + bcol] = stg[(s * B + rr) * (TW * 3) + bcol];
            }
        }
    };

    // ---- the pipeline -----------------------------------------------------------
    // iteration i: [A] store(i-1) (TMA, async) | walk(i+1) | decode(i) |
    //                  per-block dirty masks(i) | drain store(i-1) reads
    //              [B1] dirty items(i) | prefill staging with RGB(root)
    //              [B2] blend dirty items(i) into staging
    __syncthreads();
    walk(0);
    __syncthreads();
#ifdef RLFC_PHASE_TIMING
    // per-warp cycle counters: [0] store+walk, [1] decode, [2] classify masks,
    // [3] barrier A wait, [4] items+prefill, [5] barrier B1 wait, [6] blend,
    // [7] barrier B2 wait
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tc = clock64();
#define RLFC_TICK(k) do { const long long tn = clock64(); ph[k] += tn - tc; tc = tn; } while (0)
#else
#define RLFC_TICK(k) do { } while (0)
#endif
    if (P.specialized) {
        // named barriers: 1/2 row walked (parity), 3/4 row consumed (parity),
        // 5 consumer-internal.  Walkers run up to two camera rows ahead.
        if (tid >= NCONS) {
            for (int t = 1; t < T; ++t) {
                if (t >= 2) asm volatile("bar.sync %0, %1;" ::"r"(3 + (t & 1)), "r"(THREADS) : "memory");
                walk(t);
                asm volatile("bar.arrive %0, %1;" ::"r"(1 + (t & 1)), "r"(THREADS) : "memory");
            }
        } else {
            for (int i = 0; i <= T; ++i) {
                const uint64_t want = i < T ? want_mask(i) : 0ull;
                if (i >= 1 && (tid == 0 || mode != 2)) store(i - 1);
                if (i < T) {
                    if (i >= 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + (i & 1)), "r"(THREADS) : "memory");
                    decode(i);
                    classify_masks(i, want);
                }
                if (issued) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                asm volatile("bar.sync 5, %0;" ::"r"(NCONS) : "memory");
                if (i < T) {
                    classify_items(i);
                    prefill(i);
                }
                asm volatile("bar.sync 5, %0;" ::"r"(NCONS) : "memory");
                if (i < T) blend(i);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 5, %0;" ::"r"(NCONS) : "memory");
                if (i < T) asm volatile("bar.arrive %0, %1;" ::"r"(3 + (i & 1)), "r"(THREADS) : "memory");
            }
        }
    } else {
    for (int i = 0; i <= T; ++i) {
            const uint64_t want = i < T ? want_mask(i) : 0ull;   // warp-uniform per warp
            if (i >= 1 && (tid == 0 || mode != 2)) store(i - 1);
            if (i + 1 < T) walk(i + 1);
            RLFC_TICK(0);
            if (i < T) {
                decode(i);
                RLFC_TICK(1);
                classify_masks(i, want);
                RLFC_TICK(2);
            }
            if (issued) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncthreads();
            RLFC_TICK(3);
            if (i < T) {
                classify_items(i);
                prefill(i);
            }
            RLFC_TICK(4);
            __syncthreads();
            RLFC_TICK(5);
            if (i < T) blend(i);
            RLFC_TICK(6);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            RLFC_TICK(7);
        }
    }
#ifdef RLFC_PHASE_TIMING
    if ((tid & 31) == 0 && blockIdx.x < 4096) {
        for (int q = 0; q < 8; ++q) g_phase[(blockIdx.x * 8 + (tid >> 5)) * 8 + q] = ph[q];
    }
#endif
    if (issued) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
    // ---- anomaly: exact reference-order values and status ----------------------
    if (cnt[4]) tile_fallback<B>(P, by, bx0, nb, lut, nbt);
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = []() -> EncodeTiledFn {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

template <int B, int TW, typename VT, typename RT>
int launch(const rlfc_field& f, int stop_level, const int32_t* slots, int by_lo, int by_hi, uint8_t* rgb,
           int64_t img_stride, int64_t row_stride, uint64_t* status, cudaStream_t stream) {
    using C = Cfg<B, TW>;
    Params P{};
    P.f = f;
    P.stop_level = stop_level;
    P.slots = slots;
    P.by_lo = by_lo;
    P.rgb = rgb;
    P.img_stride = img_stride;
    P.row_stride = row_stride;
    P.status = status;
    P.tiles_x = (f.wb + C::NB - 1) / C::NB;
    const int h = f.tree_height, S = f.s_count;
    // level rows 1..h-1 in resl; the level-0 row (S slots) in res0
    int ns = 0;
    for (int l = 1; l < h; ++l) {
        P.slot_base[l] = ns;
        ns += f.level_sx[l];
    }
    P.ent_cap = C::NREC * (S + ns);               // every node of a row present
    const int plane = 3 * B * TW;
    const int root_row_bytes = f.rsx * plane * (int)sizeof(RT);
    P.roots_all = f.rsy * root_row_bytes <= 16 * 1024;
    P.no_prefill = 0;
#ifdef RLFC_TUNING
    // experiment knobs exist only in a tuning build (never the shipped .so)
    {
        const char* e = getenv("RLFC_TILED_NO_PREFILL");
        P.no_prefill = e && e[0] == '1';
    }
#endif
    P.roots_vec = ((f.wp * (int)sizeof(RT)) % 16) == 0 && (reinterpret_cast<uintptr_t>(f.roots) & 15) == 0;
    auto al = [](int x) { return (x + 127) & ~127; };
    int off = al((int)sizeof(DigitLut));
    P.off_nbt = off;   off = al(off + (int)sizeof(NodeBytes));
    P.off_cur = off;   off = al(off + C::NREC * MAXH * 4);
    P.off_err = off;   off = al(off + C::NREC * 4);
    P.off_cnt = off;   off = al(off + 8 * 4);
    P.off_mask = off;  off = al(off + 2 * MAXH * C::NREC * 2 * 4);
    P.seg_cap = S + ns;
    P.off_ent = off;   off = al(off + 2 * 2 * C::NREC * P.seg_cap * (int)sizeof(Entry));
    P.off_root = off;  off = al(off + (P.roots_all ? f.rsy : 1) * root_row_bytes);
    P.off_rgb = off;   off = al(off + (P.roots_all ? f.rsx * f.rsy : 1) * B * TW * 3);
    P.off_mbar = off;  off = al(off + 16);
    P.off_list = off;  off = al(off + S * C::NB * 8 + C::NB * 12);
    P.off_priv = off;  off = al(off + 2 * 2 * 2 * 32 * 4);     // prefix arrays
    P.off_res0 = off;  off = al(off + S * plane * (int)sizeof(VT));
    P.off_resl = off;  off = al(off + ns * plane * (int)sizeof(VT));
    P.off_stage = off; off = al(off + S * B * TW * 3);
    P.off_bytes = off;
    // staging window for the records: the host-measured worst tile when it
    // fits next to the other buffers, else what is left (bigger tiles take the
    // reference-order path)
    const int want = f.tile_bytes_max > 0 ? f.tile_bytes_max + 64 : 32 * 1024;
    const int cap = min(min(want, 227 * 1024 - off), 65536);   // 16-bit payload offsets
    if (cap < 4096) return RLFC_ERR_ARGUMENT;
    P.bytes_cap = cap;
    const int smem = off + cap;
    // output path
    const bool aligned = ((reinterpret_cast<uintptr_t>(rgb) | (uintptr_t)img_stride | (uintptr_t)row_stride |
                           (uintptr_t)(TW * 3)) & 15) == 0;
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    P.store_mode = aligned ? 1 : 0;
    const int nrows = min(by_hi * B, f.height) - by_lo * B;
    EncodeTiledFn enc = encode_fn();
    if (aligned && !slots && enc && S <= 256 && TW * 3 <= 256) {
        const cuuint64_t dims[4] = {(cuuint64_t)f.width * 3, (cuuint64_t)nrows, (cuuint64_t)f.t_count,
                                    (cuuint64_t)S};
        const cuuint64_t strides[3] = {(cuuint64_t)row_stride, (cuuint64_t)img_stride,
                                       (cuuint64_t)img_stride * f.t_count};
        const cuuint32_t box[4] = {(cuuint32_t)(TW * 3), (cuuint32_t)B, 1u, (cuuint32_t)S};
        const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, rgb, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
            P.store_mode = 2;
    }
    auto kern = k_decode_field_tiled<B, TW, VT, RT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int threads = 128;                               // measured best (profiles/)
    P.specialized = 0;
#ifdef RLFC_TUNING
    if (const char* e = getenv("RLFC_TILED_THREADS")) threads = atoi(e) == 256 ? 256 : 128;
    {
        // dedicated walker warps measured slower (152 vs 199 Gpix/s, cfg2 R4)
        const char* e = getenv("RLFC_TILED_SPEC");
        P.specialized = e && e[0] == '1';
        if (P.specialized) threads += 64;            // + two dedicated walker warps
    }
#endif
    const int grid = P.tiles_x * (by_hi - by_lo);
    kern<<<grid, threads, smem, stream>>>(P, map);  // P.specialized set above
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "rlfc_b200: tiled decode launch error: %s\n", cudaGetErrorString(e));
        return RLFC_ERR_CUDA;
    }
    return RLFC_OK;
}

}  // namespace tiled

#ifdef RLFC_PHASE_TIMING
extern "C" int rlfc_debug_phase(long long* host_out) {
    return cudaMemcpyFromSymbol(host_out, tiled::g_phase, sizeof(tiled::g_phase)) == cudaSuccess ? 0 : 4;
}
#endif

int launch_decode_field_tiled(const rlfc_field& f, int stop_level, const int32_t* slots, int by_lo, int by_hi,
                              uint8_t* rgb, int64_t img_stride, int64_t row_stride, uint64_t* status,
                              cudaStream_t stream) {
    using namespace tiled;
    if (f.tree_height > MAXH || f.s_count > MAXS) return RLFC_ERR_ARGUMENT;
    int nslot = f.s_count;
    for (int l = 1; l < f.tree_height; ++l) {
        if (f.level_sx[l] > 32) return RLFC_ERR_ARGUMENT;
        nslot += f.level_sx[l];
    }
    if (nslot > 64) return RLFC_ERR_ARGUMENT;       // 6-bit slot field of an Entry
    const bool small_res = f.quant_shift <= 4;      // |dequant| <= 16392 fits int16
    const bool r16 = f.roots_i16 != 0;
#define RLFC_TILED(B_, TW_)                                                                                       \
    if (small_res && r16)                                                                                         \
        return launch<B_, TW_, int16_t, int16_t>(f, stop_level, slots, by_lo, by_hi, rgb, img_stride, row_stride, \
                                                 status, stream);                                                 \
    if (small_res)                                                                                                \
        return launch<B_, TW_, int16_t, int32_t>(f, stop_level, slots, by_lo, by_hi, rgb, img_stride, row_stride, \
                                                 status, stream);                                                 \
    if (r16)                                                                                                      \
        return launch<B_, TW_, int32_t, int16_t>(f, stop_level, slots, by_lo, by_hi, rgb, img_stride, row_stride, \
                                                 status, stream);                                                 \
    return launch<B_, TW_, int32_t, int32_t>(f, stop_level, slots, by_lo, by_hi, rgb, img_stride, row_stride,     \
                                             status, stream);
    switch (f.block) {
        case 4: { RLFC_TILED(4, 32) }
        case 8: { RLFC_TILED(8, 32) }
        case 16: { RLFC_TILED(16, 16) }
        default: return RLFC_ERR_ARGUMENT;
    }
#undef RLFC_TILED
}

}  // namespace rlfc
