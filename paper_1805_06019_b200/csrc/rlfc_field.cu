// rlfc_field.cu -- fused, tiled full-field decode for sm_100a.
//
// One CTA owns one TILE: a block row `by` x NB consecutive block columns
// (TW = NB*B pixels wide), for ALL S*T views and all three channels.  The
// reference decodes view by view and re-walks every record once per view
// (kernels.py:219-242: S*T walks of each record); here every record of the
// tile is walked exactly once per launch and every present payload is
// decoded exactly once, and the per-view work is a few integer adds.
//
// Per CTA:
//   1. stage the tile's records (three contiguous byte ranges, one per
//      channel -- container.py:306-323) into shared memory with 16-byte
//      vector loads;
//   2. one thread per record pre-walks the descriptors of levels h-1..k+1 to
//      find where each tree level starts inside the record;
//   3. for every camera row t (and chunk of CH views along s):
//        walk   - one thread per record walks the level rows / level-0 chunk
//                 that row t needs (cursor per level, monotone), emitting a
//                 work item per present node (kernels.py:181-215);
//        decode - all threads BISE-decode the emitted payloads, four values
//                 per item, closed-form bit offsets, digit LUTs in smem, and
//                 store the dequantised residuals into per-node smem slots
//                 (kernels.py:128-159, 202-211);
//        blend  - a thread owns one 4-pixel quad of the tile and a pair of
//                 neighbouring views; it keeps root + levels >= 1 as a
//                 register partial sum (shared by the pair), adds the
//                 level-0 residual, applies the YCoCg-R inverse + clamp
//                 (colorspace.py:27-56) and writes RGB8 into a staging
//                 buffer; the staged rows go out as 16-byte stores.
//   Tiles whose records do not fit the staging budget, or any tile that saw
//   a stream anomaly, fall back to the reference-order per-block walk
//   (walk_chain) so values and error precedence stay exact.
#include <cuda_runtime.h>
#include <cstdio>

#include "rlfc_common.cuh"
#include "rlfc_field.cuh"

namespace rlfc {

namespace tiled {

constexpr int THREADS = 256;
constexpr int CH = 8;          // level-0 views decoded per chunk
constexpr int MAXH = 8;        // tree levels handled by the tiled kernel
constexpr int MAXROW = 32;     // max nodes in one level row (S <= 64)

struct Params {
    rlfc_field f;
    int stop_level;
    const int32_t* slots;
    int by_lo;
    uint8_t* rgb;
    int64_t img_stride, row_stride;
    uint64_t* status;
    int tiles_x;
    // smem carve (byte offsets)
    int off_nbt, off_rec, off_cur, off_err, off_mask, off_ent, off_root, off_res, off_stage, off_bytes;
    int bytes_cap, ent_cap, n_slots;
    int slot_base[MAXH];
    int vec_store;             // 1: 16-byte aligned output rows
};

// One emitted decode job: payload byte offset in the staged tile, descriptor,
// channel, destination slot and block.
struct Entry {
    uint32_t off;
    uint32_t meta;   // desc | c << 5 | blk << 7 | slot << 16
};

__device__ __forceinline__ uint32_t smem_bits32(const uint8_t* base, uint32_t bitpos) {
    const uint32_t a = bitpos >> 3;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(base + (a & ~3u));
    const uint32_t sh = ((a & 3u) << 3) + (bitpos & 7u);
    return __funnelshift_r(w[0], w[1], sh);
}

template <int B, int TW, typename VT>
struct Cfg {
    static constexpr int NB = TW / B;           // blocks per tile
    static constexpr int NREC = 3 * NB;         // records per tile
    static constexpr int BSQ = B * B;
    static constexpr int QPB = BSQ / 4;         // quads per block
    static constexpr int QPR = TW / 4;          // quads per tile row
    static constexpr int QUADS = QPR * B;       // quads per tile
    static constexpr int GROUPS = THREADS / QUADS;
    static constexpr int SLOT_VALS = 3 * NB * BSQ;
    static_assert(QUADS <= THREADS && THREADS % QUADS == 0, "tile shape");
};

// Reference-order fallback for one tile: one thread per (view, block), three
// chains walked from global memory exactly as kernels.py:162-216.  Also
// reports the exact failure key when any anomaly was seen.
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
            const uint8_t* rec = f.srv[c] + f.offsets[c][by * f.wb + bx];
            int st = walk_chain<B * B>(f, rec, s, t, P.stop_level, acc[c], lut, nb_tab);
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

// Decode values 4j..4j+3 of one payload staged in smem into the slot.
template <int BSQ, typename VT>
__device__ __forceinline__ bool decode_quad(const uint8_t* bytes, uint32_t off, int desc, int j, int shift,
                                            const DigitLut& lut, VT* dst) {
    const int mode = desc_mode(desc), b = desc_bits(desc);
    const uint32_t base = off << 3;
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = 4 * j + i;
        uint32_t z;
        if (mode == MODE_BITS) {
            z = smem_bits32(bytes, base + (uint32_t)(k * b)) & ((1u << b) - 1u);
        } else if (mode == MODE_TRIT) {
            const int g = k / 5, ii = k - 5 * g;
            const uint32_t gp = base + (uint32_t)(g * (8 + 5 * b));
            const uint32_t pack = smem_bits32(bytes, gp) & 0xFFu;
            ok &= pack <= 242u;
            const uint32_t digit = (lut.trit[pack < 243u ? pack : 0] >> (2 * ii)) & 3u;
            const uint32_t low = smem_bits32(bytes, gp + 8 + ii * b) & ((1u << b) - 1u);
            z = (digit << b) | low;
        } else {
            const int g = k / 3, ii = k - 3 * g;
            const uint32_t gp = base + (uint32_t)(g * (7 + 3 * b));
            const uint32_t pack = smem_bits32(bytes, gp) & 0x7Fu;
            ok &= pack <= 124u;
            const uint32_t digit = (lut.quint[pack < 125u ? pack : 0] >> (3 * ii)) & 7u;
            const uint32_t low = smem_bits32(bytes, gp + 7 + ii * b) & ((1u << b) - 1u);
            z = (digit << b) | low;
        }
        dst[i] = (VT)dequant(z, shift);
    }
    return ok;
}

template <int B, int TW, typename VT, typename RT>
__global__ void __launch_bounds__(THREADS, 2) k_decode_field_tiled(const Params P) {
    using C = Cfg<B, TW, VT>;
    extern __shared__ __align__(16) uint8_t smem[];
    const rlfc_field& f = P.f;
    const int tid = threadIdx.x;
    const int by = P.by_lo + blockIdx.x / P.tiles_x;
    const int tx = blockIdx.x % P.tiles_x;
    const int bx0 = tx * C::NB;
    const int nb = min(C::NB, f.wb - bx0);
    const int k = P.stop_level, h = f.tree_height;
    const int S = f.s_count, T = f.t_count;
    const int lmin = k > 0 ? k : 1;              // lowest level held as a full row

    DigitLut& lut = *reinterpret_cast<DigitLut*>(smem);
    NodeBytes& nbt = *reinterpret_cast<NodeBytes*>(smem + P.off_nbt);
    uint32_t* rec_beg = reinterpret_cast<uint32_t*>(smem + P.off_rec);
    uint32_t* cur = reinterpret_cast<uint32_t*>(smem + P.off_cur);   // [NREC][MAXH]
    int32_t* err = reinterpret_cast<int32_t*>(smem + P.off_err);     // [NREC + 2]
    uint32_t* mask = reinterpret_cast<uint32_t*>(smem + P.off_mask); // [MAXH][NREC]
    Entry* ent = reinterpret_cast<Entry*>(smem + P.off_ent);
    RT* roots = reinterpret_cast<RT*>(smem + P.off_root);            // [rsx][3][B][TW]
    VT* res = reinterpret_cast<VT*>(smem + P.off_res);               // [slot][3][B][TW]
    uint8_t* stage = smem + P.off_stage;                             // [CH][B][TW*3]
    uint8_t* bytes = smem + P.off_bytes;
    int32_t& n_ent = err[C::NREC];
    int32_t& any_err = err[C::NREC + 1];

    // ---- digit LUTs --------------------------------------------------------
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
        constexpr NodeBytes NBT = make_node_bytes<B * B>();
        if (tid < 32) nbt.v[tid] = NBT.v[tid];
    }
    // ---- stage the tile's records (three contiguous ranges) ----------------
    uint64_t beg[3], end[3], abeg[3];
    uint32_t sbase[3];
    uint32_t total = 0;
    const bool need_srv = k < h;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t blk0 = (int64_t)by * f.wb + bx0;
        beg[c] = f.offsets[c][blk0];
        end[c] = (bx0 + nb < f.wb) ? f.offsets[c][blk0 + nb]
                                   : ((by + 1 < f.hb) ? f.offsets[c][blk0 + nb] : f.srv_len[c]);
        abeg[c] = beg[c] & ~uint64_t(15);
        const uint64_t aend = (end[c] + 15) & ~uint64_t(15);
        sbase[c] = total;
        total += need_srv ? (uint32_t)(aend - abeg[c]) : 0u;
    }
    const bool fits = total + 16 <= (uint32_t)P.bytes_cap;
    __syncthreads();
    if (!fits) {
        tile_fallback<B>(P, by, bx0, nb, lut, nbt);
        return;
    }
    if (need_srv) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const uint4* src = reinterpret_cast<const uint4*>(f.srv[c] + abeg[c]);
            uint4* dst = reinterpret_cast<uint4*>(bytes + sbase[c]);
            const uint32_t n16 = (uint32_t)((((end[c] + 15) & ~uint64_t(15)) - abeg[c]) >> 4);
            for (uint32_t i = tid; i < n16; i += THREADS) dst[i] = __ldg(src + i);
        }
    }
    if (tid < C::NREC) {
        const int c = tid / C::NB, b = tid % C::NB;
        uint32_t rb = 0;
        if (b < nb) rb = sbase[c] + (uint32_t)(f.offsets[c][(int64_t)by * f.wb + bx0 + b] - abeg[c]);
        rec_beg[tid] = rb;
        err[tid] = 0;
    }
    if (tid == 0) { n_ent = 0; any_err = 0; }
    __syncthreads();

    // ---- pre-walk: where does each level start inside each record ----------
    if (tid < C::NREC && (tid % C::NB) < nb && need_srv) {
        const uint8_t* rec = bytes + rec_beg[tid];
        const uint32_t rbit = rec_beg[tid] << 3;
        uint32_t cu = (uint32_t)f.bitmap_bytes;
        uint32_t* mycur = cur + tid * MAXH;
        mycur[h - 1] = cu;
        bool bad = false;
        for (int l = h - 1; l > k && !bad; --l) {
            const int n0 = f.level_base[l], n1 = n0 + f.level_sx[l] * f.level_sy[l];
            for (int w = n0; w < n1 && !bad; w += 32) {
                uint32_t bits = smem_bits32(bytes, rbit + (uint32_t)w);
                if (n1 - w < 32) bits &= (1u << (n1 - w)) - 1u;
                while (bits) {
                    bits &= bits - 1u;
                    const int d = rec[cu];
                    if (d >= NUM_DESC) { bad = true; break; }
                    cu += nbt.v[d];
                }
            }
            mycur[l - 1] = cu;
        }
        if (bad) { err[tid] = 1; any_err = 1; }
    }
    __syncthreads();

    // thread roles for the blend: quad q (row yy, quad column xq) and group g
    const int q = tid % C::QUADS, g = tid / C::QUADS;
    const int yy = q / C::QPR, xq = q % C::QPR;
    const int blk = (xq * 4) / B;
    const bool qactive = blk < nb;
    const int rsx = f.rsx;

    for (int t = 0; t < T; ++t) {
        // root row for this camera row
        if ((t & ((1 << h) - 1)) == 0) {
            const int ry = t >> h;
            const int nval = rsx * 3 * B * TW;
            const int64_t plane = (int64_t)f.hp * f.wp;
            for (int i = tid; i < nval; i += THREADS) {
                const int x = i % TW, rr = (i / TW) % B, c = (i / (TW * B)) % 3, rx = i / (TW * B * 3);
                const int gx = bx0 * B + x;
                RT v = 0;
                if (gx < f.wp) {
                    const int64_t idx = (((int64_t)rx * f.rsy + ry) * 3 + c) * plane +
                                        (int64_t)(by * B + rr) * f.wp + gx;
                    v = reinterpret_cast<const RT*>(f.roots)[idx];
                }
                roots[i] = v;
            }
        }
        for (int s0 = 0; s0 < S; s0 += CH) {
            // skip chunks with no requested view
            bool want = false;
            for (int s = s0; s < min(S, s0 + CH); ++s) {
                const int img = s * T + t;
                if (!P.slots || P.slots[img] >= 0) want = true;
            }
            const bool rows_due = (s0 == 0);
            // ---- walk ----------------------------------------------------------
            if (tid < C::NREC && (tid % C::NB) < nb && need_srv && !err[tid]) {
                const uint8_t* rec = bytes + rec_beg[tid];
                const uint32_t rbit = rec_beg[tid] << 3;
                uint32_t* mycur = cur + tid * MAXH;
                const int c = tid / C::NB, b = tid % C::NB;
                bool bad = false;
                const int lfirst = rows_due ? h - 1 : 0;
                for (int l = lfirst; l >= 0 && !bad; --l) {
                    if (l < k) break;
                    int x0, cnt, slot0;
                    if (l >= lmin) {
                        if (!rows_due || (t & ((1 << l) - 1)) != 0) continue;
                        x0 = 0;
                        cnt = f.level_sx[l];
                        slot0 = P.slot_base[l];
                    } else {  // level 0 chunk
                        x0 = s0;
                        cnt = min(CH, S - s0);
                        slot0 = 0;
                    }
                    const int n0 = f.level_base[l] + (t >> l) * f.level_sx[l] + x0;
                    uint32_t bits = smem_bits32(bytes, rbit + (uint32_t)n0);
                    if (cnt < 32) bits &= (1u << cnt) - 1u;
                    const bool emit = (l >= lmin) || want;
                    uint32_t cu = mycur[l];
                    uint32_t mbits = bits;
                    while (bits) {
                        const int x = __ffs(bits) - 1;
                        bits &= bits - 1u;
                        const int d = rec[cu];
                        if (d >= NUM_DESC) { bad = true; break; }
                        if (emit) {
                            const int e = atomicAdd(&n_ent, 1);
                            if (e < P.ent_cap) {
                                Entry en;
                                en.off = rec_beg[tid] + cu + 1;
                                en.meta = (uint32_t)d | (uint32_t)c << 5 | (uint32_t)b << 7 |
                                          (uint32_t)(slot0 + x) << 16;
                                ent[e] = en;
                            } else {
                                bad = true;  // cannot happen with a host-sized ent_cap
                            }
                        }
                        cu += nbt.v[d];
                    }
                    mycur[l] = cu;
                    mask[l * C::NREC + tid] = mbits;
                }
                if (bad) { err[tid] = 1; any_err = 1; }
            }
            __syncthreads();
            // ---- decode --------------------------------------------------------
            const int ne = min(n_ent, P.ent_cap);
            for (int it = tid; it < ne * C::QPB; it += THREADS) {
                const int e = it / C::QPB, j = it - e * C::QPB;
                const Entry en = ent[e];
                const int d = en.meta & 31, c = (en.meta >> 5) & 3, b = (en.meta >> 7) & 511;
                const int slot = en.meta >> 16;
                const int row = (4 * j) / B, col = (4 * j) % B;
                VT* dst = res + (((size_t)slot * 3 + c) * B + row) * TW + b * B + col;
                if (!decode_quad<C::BSQ, VT>(bytes, en.off, d, j, f.quant_shift, lut, dst)) {
                    err[c * C::NB + b] = 1;
                    any_err = 1;
                }
            }
            __syncthreads();
            if (tid == 0) n_ent = 0;
            // ---- blend + store ---------------------------------------------------
            if (want && !any_err) {
                for (int p = g; p < CH / 2; p += C::GROUPS) {
                    const int sa = s0 + 2 * p;
                    if (sa >= S || !qactive) continue;
                    int32_t acc[3][4];
                    const int rx = sa >> h;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const RT* rp = roots + ((rx * 3 + c) * B + yy) * TW + xq * 4;
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[c][i] = (int32_t)rp[i];
                    }
                    for (int l = h - 1; l >= lmin; --l) {
                        const int x = sa >> l;
                        const int slot = P.slot_base[l] + x;
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            if ((mask[l * C::NREC + c * C::NB + blk] >> x) & 1u) {
                                const VT* rp = res + (((size_t)slot * 3 + c) * B + yy) * TW + xq * 4;
#pragma unroll
                                for (int i = 0; i < 4; ++i) acc[c][i] += (int32_t)rp[i];
                            }
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int s = sa + e;
                        if (s >= S) break;
                        int32_t v[3][4];
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
#pragma unroll
                            for (int i = 0; i < 4; ++i) v[c][i] = acc[c][i];
                            if (k == 0) {
                                const int x = s - s0;
                                if ((mask[c * C::NB + blk] >> x) & 1u) {
                                    const VT* rp = res + (((size_t)x * 3 + c) * B + yy) * TW + xq * 4;
#pragma unroll
                                    for (int i = 0; i < 4; ++i) v[c][i] += (int32_t)rp[i];
                                }
                            }
                        }
                        uint32_t w[3] = {0, 0, 0};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            uint32_t r, gg, bb;
                            ycocg_to_rgb8(v[0][i], v[1][i], v[2][i], r, gg, bb);
                            const int byte = 3 * i;
                            w[byte >> 2] |= r << (8 * (byte & 3));
                            w[(byte + 1) >> 2] |= gg << (8 * ((byte + 1) & 3));
                            w[(byte + 2) >> 2] |= bb << (8 * ((byte + 2) & 3));
                        }
                        uint32_t* sp = reinterpret_cast<uint32_t*>(stage + ((s - s0) * B + yy) * (TW * 3) + xq * 12);
                        sp[0] = w[0];
                        sp[1] = w[1];
                        sp[2] = w[2];
                    }
                }
                __syncthreads();
                // store the staged rows of every requested view in the chunk
                const int row_bytes = min(TW, f.width - bx0 * B) * 3;
                if (row_bytes > 0) {
                    const int nvec = (TW * 3) / 16;
                    const int items = CH * B * nvec;
                    for (int it = tid; it < items; it += THREADS) {
                        const int v16 = it % nvec, rr = (it / nvec) % B, sl = it / (nvec * B);
                        const int s = s0 + sl;
                        const int y = by * B + rr;
                        if (s >= S || y >= f.height) continue;
                        const int img = s * T + t;
                        const int slot = P.slots ? P.slots[img] : img;
                        if (slot < 0) continue;
                        uint8_t* orow = P.rgb + (int64_t)slot * P.img_stride +
                                        (int64_t)(y - P.by_lo * B) * P.row_stride + (int64_t)bx0 * B * 3;
                        const uint8_t* src = stage + (sl * B + rr) * (TW * 3);
                        const int b0 = v16 * 16;
                        if (P.vec_store && b0 + 16 <= row_bytes) {
                            *reinterpret_cast<uint4*>(orow + b0) = *reinterpret_cast<const uint4*>(src + b0);
                        } else {
                            for (int bb = b0; bb < min(b0 + 16, row_bytes); ++bb) orow[bb] = src[bb];
                        }
                    }
                }
            }
            __syncthreads();
        }
    }
    // ---- anomaly: exact reference-order status (and values) ----------------
    if (any_err) {
        __syncthreads();
        tile_fallback<B>(P, by, bx0, nb, lut, nbt);
    }
}

template <int B, int TW, typename VT, typename RT>
int launch(const rlfc_field& f, int stop_level, const int32_t* slots, int by_lo, int by_hi, uint8_t* rgb,
           int64_t img_stride, int64_t row_stride, uint64_t* status, cudaStream_t stream) {
    using C = Cfg<B, TW, VT>;
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
    const int h = f.tree_height;
    // slots: level-0 chunk [0, CH), then full rows of levels 1..h-1
    int ns = CH;
    for (int l = 1; l < h; ++l) {
        P.slot_base[l] = ns;
        ns += f.level_sx[l];
    }
    P.slot_base[0] = 0;
    P.n_slots = ns;
    int row_nodes = CH;
    for (int l = 1; l < h; ++l) row_nodes += f.level_sx[l];
    P.ent_cap = C::NREC * row_nodes;
    auto al = [](int x) { return (x + 15) & ~15; };
    int off = al((int)sizeof(DigitLut));
    P.off_nbt = off;   off = al(off + (int)sizeof(NodeBytes));
    P.off_rec = off;   off = al(off + C::NREC * 4);
    P.off_cur = off;   off = al(off + C::NREC * MAXH * 4);
    P.off_err = off;   off = al(off + (C::NREC + 2) * 4);
    P.off_mask = off;  off = al(off + MAXH * C::NREC * 4);
    P.off_ent = off;   off = al(off + P.ent_cap * (int)sizeof(Entry));
    P.off_root = off;  off = al(off + f.rsx * 3 * B * TW * (int)sizeof(RT));
    P.off_res = off;   off = al(off + ns * C::SLOT_VALS * (int)sizeof(VT));
    P.off_stage = off; off = al(off + CH * B * TW * 3);
    P.off_bytes = off;
    const int budget = 113 * 1024;                  // two CTAs per SM
    int cap = budget - off;
    if (cap < 16 * 1024) cap = 16 * 1024;           // keep a useful window; 1 CTA/SM then
    P.bytes_cap = cap;
    const int smem = off + cap;
    if (smem > 227 * 1024) return RLFC_ERR_ARGUMENT;
    P.vec_store = ((reinterpret_cast<uintptr_t>(rgb) | (uintptr_t)img_stride | (uintptr_t)row_stride) & 15) == 0;
    auto kern = k_decode_field_tiled<B, TW, VT, RT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = P.tiles_x * (by_hi - by_lo);
    kern<<<grid, THREADS, smem, stream>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "rlfc_b200: tiled decode launch error: %s\n", cudaGetErrorString(e));
        return RLFC_ERR_CUDA;
    }
    return RLFC_OK;
}

}  // namespace tiled

int launch_decode_field_tiled(const rlfc_field& f, int stop_level, const int32_t* slots, int by_lo, int by_hi,
                              uint8_t* rgb, int64_t img_stride, int64_t row_stride, uint64_t* status,
                              cudaStream_t stream) {
    using namespace tiled;
    // envelope of the tiled kernel
    if (f.tree_height > MAXH || f.s_count > 64) return RLFC_ERR_ARGUMENT;
    for (int l = 1; l < f.tree_height; ++l)
        if (f.level_sx[l] > MAXROW) return RLFC_ERR_ARGUMENT;
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
        case 4: { RLFC_TILED(4, 64) }
        case 8: { RLFC_TILED(8, 64) }
        case 16: { RLFC_TILED(16, 32) }
        default: return RLFC_ERR_ARGUMENT;
    }
#undef RLFC_TILED
}

}  // namespace rlfc
