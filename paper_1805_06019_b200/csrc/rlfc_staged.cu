// rlfc_staged.cu -- staged full-field decode (sm_100a): index -> payloads -> blend.
//
// The reference decodes image by image and re-walks every record once per
// image (decoder.py:187-210 -> kernels.py:219-242 -> decode_chain_core
// kernels.py:162-216).  Here the work is split into launches, each with
// full-warp parallelism and no per-camera-row barriers:
//
//   k_root_rgb  RGB8 of every root sample of the band (colorspace.py:27-56).
//   k_index     one lane per record (channel, block): popcount of the
//               presence bitmap (kernels.py:181-183) reserves a dense run of
//               payload slots (one atomic per warp), then the lane walks the
//               descriptors (kernels.py:185-200) and writes one entry per
//               present node (payload byte offset, descriptor, channel,
//               block), plus the record's bitmap words and per-word slot
//               ranks into word-major tables.  Records with any anomaly are
//               flagged.
//   k_payloads  one lane per payload, CTAs bucket 512 entries by BISE mode
//               so every warp runs one unrolled code path
//               (kernels.py:128-159); for B = 4 the chunk's contiguous SRV
//               bytes are staged in shared memory (double-buffered, cp.async)
//               and each group is one 64-bit window at its closed-form bit
//               offset; dequantisation (kernels.py:202-211) is a table.  A
//               corrupt pack flags its record.
//   k_blend     one 128-thread CTA per (column chunk of 64 pixels, camera
//               row, block row), all S views.  The last warp issues TMA
//               tensor loads of every view's RGB(root) rows (the result for
//               clean pixels) and of the raw roots; the record phase reads
//               row masks and slot bases from the word-major tables; one
//               thread per (view, block) pair finds the dirty pairs and
//               appends them (warp-aggregated atomics); tasks add the
//               present residuals (16-byte gathers), YCoCg-R inverse + clamp
//               + pack over the prefilled bytes; TMA tensor stores write the
//               staged rows straight to HBM.  (view, block) pairs touching a
//               flagged record run the reference-order walk (walk_chain),
//               which reproduces the reference's values and failure order.
//
// Workspace (caller-owned device memory, rlfc_decode_workspace_bytes):
//   u64 counters | u32 rec_base[3*nblk] | u32 rec_flag[3*nblk] |
//   uint2 entries[cap] | VT residuals[cap][B*B] (VT int16 when the
//   quantisation shift keeps |residual| <= 16392, else int32) |
//   RGB8 root colours | word-major bitmap words and word ranks.
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rlfc_common.cuh"
#include "rlfc_field.cuh"

namespace rlfc {
namespace staged {

constexpr int MAXH = 8;
constexpr int MAXS = 64;
constexpr int THREADS = 256;
constexpr uint32_t SKIP = 31;       // entry descriptor: slot not decoded
constexpr int SEL_MAX = SEL_NODES_MAX;         // slot-mode decodes needing at most this many chain nodes decode only those
constexpr int STRIP = 64;           // pixels per TMA box column (192 bytes)

__device__ const DigitLut g_lut = make_digit_lut();
__device__ const NodeBytes g_nb4 = make_node_bytes<16>();
__device__ const NodeBytes g_nb8 = make_node_bytes<64>();
__device__ const NodeBytes g_nb16 = make_node_bytes<256>();

template <int BSQ>
__device__ __forceinline__ const NodeBytes& node_bytes() {
    return BSQ == 16 ? g_nb4 : BSQ == 64 ? g_nb8 : g_nb16;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Ws {
    unsigned long long* counter;
    uint32_t* rec_base;
    uint32_t* rec_flag;
    uint2* entries;
    uint2* sorted;         // [cap rounded to PAY_CHUNK] entries of each 512-slot chunk ordered by BISE mode
    void* res;
    uint8_t* root_rgb;     // RGB8 of every root sample, rows of rgb_stride bytes
    int rgb_stride;
    uint32_t* bm;          // [nwp][3*nblk] record bitmaps as aligned 32-bit words (word-major:
                           // one level row's words of consecutive records are contiguous)
    uint32_t* rk;          // [nwp][3*nblk] slot of the first present node of each word
    uint32_t* flist;       // [3*nblk + 1] records with a stream anomaly (prepare-time), count first
    uint32_t* units;       // [tile][1 + ucap] prepared dirty-unit lists of the B = 4 blend (count first)
    uint32_t* sel;         // [1 + SEL_MAX] chain nodes of a slot-mode decode (count first)
    int ucap;
    int nwp;
    uint64_t cap;
};

static uint64_t al256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

static int value_bytes(const rlfc_field& f) { return f.quant_shift <= 4 ? 2 : 4; }

// Carve the workspace; returns the bytes needed for `cap` payload slots.
static uint64_t carve(const rlfc_field& f, void* base, uint64_t cap, Ws* w) {
    const uint64_t nrec = 3ull * (uint64_t)f.wb * (uint64_t)f.hb;
    const uint64_t bsq = (uint64_t)f.block * (uint64_t)f.block;
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t o = off;
        off = al256(off + bytes);
        return o;
    };
    const int rgb_stride = (f.wp * 3 + 15) & ~15;
    const int nwp = (f.m_nodes + 31) / 32 + 2;
    const uint64_t o_cnt = take(8), o_base = take(4 * nrec), o_flag = take(4 * nrec), o_ent = take(8 * cap),
                   o_sort = take(8 * ((cap + 511) / 512) * 512),
                   o_res = take(cap * bsq * (uint64_t)value_bytes(f)),
                   o_rgb = take((uint64_t)f.rsx * f.rsy * f.hp * (uint64_t)rgb_stride),
                   o_bm = take(4 * nrec * (uint64_t)nwp), o_rk = take(4 * nrec * (uint64_t)nwp),
                   o_fl = take(4 * (nrec + 1));
    // prepared dirty-unit lists (B = 4, 64-pixel blend tiles, h <= 6): per
    // tile (block row, camera row, chunk) a count and up to S * 16 entries
    const bool ul = f.block == 4 && f.tree_height <= 6;
    const uint64_t ucap = (uint64_t)f.s_count * 16;
    const uint64_t ntiles = (uint64_t)f.hb * f.t_count * ((f.wb + 15) / 16);
    const uint64_t o_ul = take(ul ? 4 * ntiles * (1 + ucap) : 0);
    const uint64_t o_sel = take(4 * (1 + SEL_MAX));
    if (w) {
        uint8_t* b = static_cast<uint8_t*>(base);
        w->counter = reinterpret_cast<unsigned long long*>(b + o_cnt);
        w->rec_base = reinterpret_cast<uint32_t*>(b + o_base);
        w->rec_flag = reinterpret_cast<uint32_t*>(b + o_flag);
        w->entries = reinterpret_cast<uint2*>(b + o_ent);
        w->sorted = reinterpret_cast<uint2*>(b + o_sort);
        w->res = b + o_res;
        w->root_rgb = b + o_rgb;
        w->rgb_stride = rgb_stride;
        w->bm = reinterpret_cast<uint32_t*>(b + o_bm);
        w->rk = reinterpret_cast<uint32_t*>(b + o_rk);
        w->flist = reinterpret_cast<uint32_t*>(b + o_fl);
        w->units = ul ? reinterpret_cast<uint32_t*>(b + o_ul) : nullptr;
        w->sel = reinterpret_cast<uint32_t*>(b + o_sel);
        w->ucap = (int)ucap;
        w->nwp = nwp;
        w->cap = cap;
    }
    return off;
}

// Record (c, blk) bounds: [off, end) inside channel c's SRV section, or false
// when the offsets are inconsistent or the bitmap does not fit.
__device__ __forceinline__ bool record_span(const rlfc_field& f, int c, int64_t blk, uint64_t& off,
                                            uint64_t& len) {
    const int64_t nblk = (int64_t)f.wb * f.hb;
    off = f.offsets[c][blk];
    const uint64_t end = blk + 1 < nblk ? f.offsets[c][blk + 1] : f.srv_len[c];
    if (off > end || end > f.srv_len[c] || end - off < (uint64_t)f.bitmap_bytes) return false;
    len = end - off;
    return true;
}

// Present nodes among [0, n) of a record bitmap.
__device__ __forceinline__ uint32_t popc_prefix(const uint8_t* rec, int n) {
    uint32_t cnt = 0;
    int n0 = 0;
    for (; n0 + 32 <= n; n0 += 32) cnt += __popc(bitmap_word(rec, n0));
    if (n0 < n) cnt += __popc(bitmap_word(rec, n0) & ((1u << (n - n0)) - 1u));
    return cnt;
}

// ---- presence count (workspace sizing) -----------------------------------------
__global__ void k_count_present(const __grid_constant__ rlfc_field f, unsigned long long* out) {
    const int64_t nblk = (int64_t)f.wb * f.hb;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t n = 0;
    if (i < 3 * nblk) {
        const int c = (int)(i / nblk);
        const int64_t blk = i % nblk;
        uint64_t off, len;
        if (record_span(f, c, blk, off, len)) n = popc_prefix(f.srv[c] + off, f.m_nodes);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(out, (unsigned long long)n);
}

// ---- prepared index: per-record present counts and their exclusive prefix ---------------
__global__ void k_rec_count(const __grid_constant__ rlfc_field f, uint32_t* cnt) {
    const int64_t nblk = (int64_t)f.wb * f.hb;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * nblk) return;
    const int c = (int)(i / nblk);
    const int64_t blk = i % nblk;
    uint64_t off, len;
    cnt[i] = record_span(f, c, blk, off, len) ? popc_prefix(f.srv[c] + off, f.m_nodes) : 0u;
}

// In-place exclusive scan of n counts by one CTA of 1024 threads (each thread
// a contiguous run); the total goes to *total.  Init-time only.
__global__ void __launch_bounds__(1024) k_scan_bases(uint32_t* v, int64_t n, unsigned long long* total) {
    __shared__ unsigned long long part[1024];
    const int tid = threadIdx.x;
    const int64_t per = (n + 1023) / 1024, lo = tid * per, hi = min(n, lo + per);
    unsigned long long sum = 0;
    for (int64_t i = lo; i < hi; ++i) sum += v[i];
    part[tid] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const unsigned long long y = tid >= o ? part[tid - o] : 0ull;
        __syncthreads();
        part[tid] += y;
        __syncthreads();
    }
    unsigned long long run = part[tid] - sum;
    for (int64_t i = lo; i < hi; ++i) {
        const uint32_t x = v[i];
        v[i] = (uint32_t)run;
        run += x;
    }
    if (tid == 1023) *total = part[1023];
}

// Record slot bases for many records: per-CTA sums of 4096 counts
// (k_scan_part), an exclusive scan of those sums (k_scan_bases on the
// partials), then each CTA's in-place exclusive scan offset by its partial
// (k_scan_apply).  A single CTA walking 196,608 counts took 0.39 ms.
constexpr int SCAN_TILE = 4096;
__global__ void __launch_bounds__(256) k_scan_part(const uint32_t* v, int64_t n, uint32_t* part) {
    __shared__ uint32_t ws[8];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < SCAN_TILE / 256; ++j) {
        const int64_t i = base + j * 256 + threadIdx.x;
        if (i < n) sum += v[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 8; ++w) t += ws[w];
        part[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) k_scan_apply(uint32_t* v, int64_t n, const uint32_t* part) {
    __shared__ uint32_t ws[8];
    constexpr int PER = SCAN_TILE / 256;
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * PER;
    uint32_t x[PER];
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        x[j] = base + j < n ? v[base + j] : 0u;
        sum += x[j];
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    uint32_t run = part[blockIdx.x] + incl - sum;
    for (int w = 0; w < wid; ++w) run += ws[w];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        if (base + j < n) v[base + j] = run;
        run += x[j];
    }
}

// ---- pass 1: index -----------------------------------------------------------------
// Records whose bitmap fits IDX_MAXW - 4 aligned words (bitmap_bytes <= 64,
// e.g. M = 395 -> 50 bytes) load it once with aligned 16-byte loads, all in
// flight together, and take the popcount and the blend's word tables from
// registers: the per-lane bitmap reads (every warp load touching 32 lines)
// were most of k_index's time.
constexpr int IDX_MAXW = 20;
__device__ __forceinline__ uint32_t node_word(const uint32_t* A, int j, uint32_t sh, int node_end) {
    const int n0 = 32 * j;
    if (n0 >= node_end) return 0u;
    uint32_t v = __funnelshift_r(A[j], A[j + 1], sh);
    if (node_end - n0 < 32) v &= (1u << (node_end - n0)) - 1u;
    return v;
}

// Levels >= k occupy serial nodes [0, node_end) (level h-1 first,
// container.py:102-145); only those are indexed and decoded.
template <int BSQ>
__global__ void __launch_bounds__(THREADS) k_index(const __grid_constant__ rlfc_field f, int k, int by_lo,
                                                   int by_hi, Ws w, const uint32_t* base_in) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");      // k_root_rgb may run alongside
    const int64_t nblk = (int64_t)f.wb * f.hb;
    const int64_t band = (int64_t)(by_hi - by_lo) * f.wb;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = i < 3 * band;
    const int c = valid ? (int)(i / band) : 0;
    const int64_t blk = valid ? (int64_t)by_lo * f.wb + i % band : 0;
    const int node_end = f.level_base[k] + f.level_sx[k] * f.level_sy[k];
    uint64_t off = 0, len = 0;
    uint32_t flag = 0, count = 0;
    const bool fastbm = f.bitmap_bytes + 15 + 4 <= IDX_MAXW * 4;
    uint32_t A[IDX_MAXW];
#pragma unroll
    for (int j = 0; j < IDX_MAXW; ++j) A[j] = 0u;
    uint32_t sh = 0;
    int w0 = 0;                               // first aligned word of the bitmap in A
    if (valid) {
        if (record_span(f, c, blk, off, len)) {
            if (fastbm) {
                const uintptr_t ra = reinterpret_cast<uintptr_t>(f.srv[c] + off);
                const uint4* a = reinterpret_cast<const uint4*>(ra & ~uintptr_t(15));
                const uint32_t lead = (uint32_t)(ra & 15u);
                const int nq = (int)((lead + (uint32_t)f.bitmap_bytes + 15u) >> 4);
#pragma unroll
                for (int q = 0; q < IDX_MAXW / 4; ++q)
                    if (q < nq) {
                        const uint4 v = __ldg(a + q);
                        A[4 * q] = v.x; A[4 * q + 1] = v.y; A[4 * q + 2] = v.z; A[4 * q + 3] = v.w;
                    }
                // shift the words down so A[0] holds the bitmap's first byte's word
                w0 = (int)(lead >> 2);
#pragma unroll
                for (int j = 0; j < IDX_MAXW; ++j) {
                    const uint32_t x1 = j + 1 < IDX_MAXW ? A[j + 1] : 0u, x2 = j + 2 < IDX_MAXW ? A[j + 2] : 0u,
                                   x3 = j + 3 < IDX_MAXW ? A[j + 3] : 0u;
                    A[j] = w0 == 0 ? A[j] : w0 == 1 ? x1 : w0 == 2 ? x2 : x3;
                }
                sh = (uint32_t)(ra & 3u) * 8u;
#pragma unroll
                for (int j = 0; j + 1 < IDX_MAXW - 3; ++j) count += __popc(node_word(A, j, sh, node_end));
            } else {
                count = popc_prefix(f.srv[c] + off, node_end);
            }
        } else {
            flag = 1;
        }
    }
    // dense slot run per record: warp scan + one atomic per warp
    const int lane = threadIdx.x & 31;
    uint32_t incl = count;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    uint64_t slot0;
    if (base_in) {
        // prepared index: record slot bases are the exclusive prefix of the
        // records' present counts in record order (k_scan_bases)
        if (!valid) return;
        slot0 = base_in[(int64_t)c * nblk + blk];
    } else {
        unsigned long long wbase = 0;
        if (lane == 31 && incl) wbase = atomicAdd(w.counter, (unsigned long long)incl);
        wbase = __shfl_sync(0xffffffffu, wbase, 31);
        slot0 = wbase + incl - count;
        if (!valid) return;
    }
    if (slot0 + count > w.cap) flag = 1;
    const int64_t ri = (int64_t)c * nblk + blk;
    if (fastbm && !flag) {
        // bitmap words of levels >= k and the slot at each word start, for
        // the blend's row masks and ranks (k_blend); a record the walk then
        // flags never has its words read
        const int64_t nrec = 3 * nblk;
        uint32_t run = (uint32_t)slot0;
#pragma unroll
        for (int wi = 0; wi + 1 < IDX_MAXW - 3; ++wi) {
            if (wi < w.nwp) {
                const uint32_t word = node_word(A, wi, sh, node_end);
                w.bm[wi * nrec + ri] = word;
                w.rk[wi * nrec + ri] = run;
                run += __popc(word);
            }
        }
        for (int wi = IDX_MAXW - 4; wi < w.nwp; ++wi) {
            w.bm[wi * nrec + ri] = 0u;
            w.rk[wi * nrec + ri] = run;
        }
    }
    uint32_t rank = 0;
    if (!flag && count) {
        const uint8_t* rec = f.srv[c] + off;
        const NodeBytes& nb = node_bytes<BSQ>();
        uint32_t cursor = (uint32_t)f.bitmap_bytes;
        // The present nodes of [0, node_end) are the record's first `count`
        // nodes in stream order (BFS puts levels >= k first), so the walk is
        // one flat loop of `count` hops: a warp runs max-over-lanes hops, not
        // the sum over bitmap words of per-word maxima.
        // entries go out as full 32-byte sectors: slots of an aligned quad are
        // held in registers until its last slot exists (one 256-bit store);
        // partial quads at the run's ends are stored entry by entry
        uint2 p0 = make_uint2(0u, 0u), p1 = p0, p2 = p0;
        uint32_t pm = 0;                                // pending quad positions
        uint64_t pq = 0;                                // their quad's first slot
        auto flush = [&]() {
            if (pm & 1u) w.entries[pq] = p0;
            if (pm & 2u) w.entries[pq + 1] = p1;
            if (pm & 4u) w.entries[pq + 2] = p2;
            pm = 0;
        };
        for (; rank < count; ++rank) {
            const int d = cursor < len ? rec[cursor] : NUM_DESC;
            if (d >= NUM_DESC) {
                flag = 1;
                break;
            }
            const uint32_t sz = BSQ == 16 ? node_bytes16(d) : (uint32_t)nb.v[d];
            if (cursor + sz > len) {
                flag = 1;
                break;
            }
            const uint2 e = make_uint2((uint32_t)(off + cursor + 1), (uint32_t)d | (uint32_t)c << 5 | (uint32_t)blk << 7);
            const uint64_t sl = slot0 + rank;
            const uint32_t pos = (uint32_t)sl & 3u;
            pq = sl - pos;
            if (pos == 0) { p0 = e; pm |= 1u; }
            else if (pos == 1) { p1 = e; pm |= 2u; }
            else if (pos == 2) { p2 = e; pm |= 4u; }
            else if (pm == 7u) {
                asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(w.entries + pq),
                             "r"(p0.x), "r"(p0.y), "r"(p1.x), "r"(p1.y), "r"(p2.x), "r"(p2.y), "r"(e.x), "r"(e.y)
                             : "memory");
                pm = 0;
            } else {
                flush();
                w.entries[sl] = e;
            }
            cursor += sz;
        }
        flush();
    }
    // every reserved slot below the capacity is written (SKIP when not decoded)
    for (uint64_t r = rank; r < count && slot0 + r < w.cap; ++r) w.entries[slot0 + r] = make_uint2(0u, SKIP);
    if (!fastbm && !flag) {
        // bitmap words of levels >= k and the slot at each word start, for
        // the blend's row masks and ranks (k_blend)
        const uint8_t* rec = f.srv[c] + off;
        const int64_t nrec = 3 * nblk;
        uint32_t run = (uint32_t)slot0;
        for (int wi = 0; wi < w.nwp; ++wi) {
            const int n0 = wi * 32;
            uint32_t word = 0;
            if (n0 < node_end) {
                word = bitmap_word(rec, n0);
                if (node_end - n0 < 32) word &= (1u << (node_end - n0)) - 1u;
            }
            w.bm[wi * nrec + ri] = word;
            w.rk[wi * nrec + ri] = run;
            run += __popc(word);
        }
    }
    w.rec_flag[ri] = flag;
    w.rec_base[ri] = (uint32_t)slot0;
}

// ---- pass 2: payloads ----------------------------------------------------------------
// Sequential LSB-first bit reader over a byte address (kernels.py:1-11 bit
// order); reads at most 8 bytes past the last consumed bit (device SRV copies
// carry 16 bytes of zero padding).
struct BitReader {
    const uint32_t* w;
    uint64_t buf;
    uint32_t n;
    __device__ __forceinline__ explicit BitReader(const uint8_t* p) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p);
        w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
        const uint32_t sh = (uint32_t)(a & 3) * 8u;
        buf = ((uint64_t)__ldg(w) | (uint64_t)__ldg(w + 1) << 32) >> sh;
        n = 64u - sh;
        w += 2;
    }
    __device__ __forceinline__ uint32_t get(uint32_t k) {     // k <= 11
        if (n < 32u) {
            buf |= (uint64_t)__ldg(w) << n;
            ++w;
            n += 32u;
        }
        const uint32_t v = (uint32_t)buf & ((1u << k) - 1u);
        buf >>= k;
        n -= k;
        return v;
    }
};

template <typename VT>
__device__ __forceinline__ void store4(VT* p, const int32_t* v);
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
template <typename VT>
__device__ __forceinline__ void add4(const VT* p, int32_t* v);
template <>
__device__ __forceinline__ void add4<int16_t>(const int16_t* p, int32_t* v) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
    v[0] += (int32_t)(int16_t)(w.x & 0xFFFFu);
    v[1] += (int32_t)w.x >> 16;
    v[2] += (int32_t)(int16_t)(w.y & 0xFFFFu);
    v[3] += (int32_t)w.y >> 16;
}
template <>
__device__ __forceinline__ void add4<int32_t>(const int32_t* p, int32_t* v) {
    const int4 w = __ldg(reinterpret_cast<const int4*>(p));
    v[0] += w.x; v[1] += w.y; v[2] += w.z; v[3] += w.w;
}

template <typename VT>
__device__ __forceinline__ void add8(const VT* p, int32_t* v);
template <>
__device__ __forceinline__ void add8<int16_t>(const int16_t* p, int32_t* v) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] += (int32_t)(int16_t)(x[i] & 0xFFFFu);
        v[2 * i + 1] += (int32_t)x[i] >> 16;
    }
}
template <>
__device__ __forceinline__ void add8<int32_t>(const int32_t* p, int32_t* v) {
    const int4 a = __ldg(reinterpret_cast<const int4*>(p)), b = __ldg(reinterpret_cast<const int4*>(p) + 1);
    v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
    v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
}

// NV consecutive values of one payload starting at a group boundary, fully
// unrolled for a compile-time mode: groups of G values behind a PB-bit pack
// (plain bits: G = 1, PB = 0), kernels.py:128-159 bit layout.
template <int G, int PB, int NV, typename VT>
__device__ __forceinline__ void decode_run(BitReader& br, const uint16_t* lut, uint32_t b, int shift, VT* out,
                                           bool& bad) {
    constexpr uint32_t DB = G == 5 ? 2u : 3u, DMASK = G == 5 ? 3u : 7u, PMAX = G == 5 ? 242u : 124u;
    uint32_t digits = 0;
    int32_t v[4];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        if (PB && k % G == 0) {
            const uint32_t pk = br.get(PB);
            bad |= pk > PMAX;
            digits = lut[pk <= PMAX ? pk : 0u];
        }
        const uint32_t low = br.get(b);
        const uint32_t z = PB ? ((((digits >> (DB * (uint32_t)(k % G))) & DMASK) << b) | low) : low;
        v[k & 3] = deq(z, shift);
        if ((k & 3) == 3) store4<VT>(out + (k & ~3), v);
    }
}

template <int G, int PB, int BSQ, typename VT>
__device__ __forceinline__ bool decode_payload(const uint8_t* p, const uint16_t* lut, uint32_t b, int shift,
                                               VT* out) {
    constexpr int CH = 4 * G;                        // values per unrolled chunk (group- and quad-aligned)
    BitReader br(p);
    bool bad = false;
#pragma unroll 1
    for (int q = 0; q + CH <= BSQ; q += CH) decode_run<G, PB, CH, VT>(br, lut, b, shift, out + q, bad);
    if constexpr (BSQ % CH != 0) decode_run<G, PB, BSQ % CH, VT>(br, lut, b, shift, out + BSQ - BSQ % CH, bad);
    return bad;
}

// B = 4 (16 values, <= 176 payload bits): the payload's aligned words are
// read from the chunk's staged SRV bytes in shared memory; each BISE group
// (or plain-bit quad) is one
// 64-bit window at its closed-form bit offset (every group but the last is
// full), so all reads of a payload are independent;
// dequantisation is a table lookup (z < 2048 for every descriptor).

// 16-byte store with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void st16_hint(void* p, uint32_t x, uint32_t y, uint32_t z, uint32_t w, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(x), "r"(y), "r"(z),
                 "r"(w), "l"(pol)
                 : "memory");
}

template <int MODE, typename VT>
__device__ __forceinline__ bool decode16(const uint32_t* sw, uint32_t bit0, uint32_t b, const uint16_t* dlut,
                                         const VT* dq, VT* out, uint64_t pol = 0) {
    const uint32_t lm = (1u << b) - 1u;
    int32_t v[16];
    bool bad = false;
    if (MODE == MODE_BITS) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t w = win64(sw, bit0 + 4u * (uint32_t)q * b);
#pragma unroll
            for (int i = 0; i < 4; ++i) v[4 * q + i] = dq[(uint32_t)(w >> ((uint32_t)i * b)) & lm];
        }
    } else {
        constexpr int G = MODE == MODE_TRIT ? 5 : 3, PB = MODE == MODE_TRIT ? 8 : 7;
        constexpr uint32_t DB = MODE == MODE_TRIT ? 2u : 3u, DMASK = MODE == MODE_TRIT ? 3u : 7u;
        constexpr uint32_t PMAX = MODE == MODE_TRIT ? 242u : 124u;
        const uint32_t gbits = PB + G * b;
#pragma unroll
        for (int g = 0; g * G < 16; ++g) {
            const uint64_t w = win64(sw, bit0 + (uint32_t)g * gbits);
            const uint32_t pk = (uint32_t)w & ((1u << PB) - 1u);
            bad |= pk > PMAX;
            const uint32_t dg = dlut[pk <= PMAX ? pk : 0u];
#pragma unroll
            for (int i = 0; i < G && g * G + i < 16; ++i) {
                const uint32_t low = (uint32_t)(w >> (PB + (uint32_t)i * b)) & lm;
                v[g * G + i] = dq[(((dg >> (DB * i)) & DMASK) << b) | low];
            }
        }
    }
    if (sizeof(VT) == 2 && pol) {
        // int16 residuals: two 16-byte stores that stay in L2 for k_blend's gathers
        uint32_t u[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) u[q] = ((uint32_t)v[2 * q] & 0xFFFFu) | ((uint32_t)v[2 * q + 1] << 16);
        // one 256-bit store: the payload's whole 32-byte sector
        asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(out),
                     "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]),
                     "l"(pol)
                     : "memory");
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) store4<VT>(out + 4 * q, v + 4 * q);
    }
    return bad;
}

// Payload decode over the prepared index.  Slots form chunks of PAY_CHUNK
// consecutive payloads (consecutive nodes of consecutive records: one
// contiguous SRV byte range per channel), and rlfc_staged_prepare stores each
// chunk's entries ordered by BISE mode (k_sort_chunks), so a warp runs one
// mode's unrolled code (kernels.py:128-159).  A CTA takes chunks of the
// band's slot ranges, software-pipelined: while chunk i decodes, chunk i+1's
// entries are in registers and its SRV byte range is on its way into the
// other shared buffer (cp.async).  Dequantisation (kernels.py:202-211) is a
// table.  A corrupt pack flags its record (kernels.py:147-150).
constexpr int PAY_CHUNK = 512;
constexpr int PAY_BUF = 12 * 1024;       // staged SRV bytes per chunk (two buffers, dynamic shared memory)

// record of a payload slot (slot bases ascend in record order)
__device__ int64_t record_of_slot(const uint32_t* rec_base, int64_t nrec, uint64_t slot) {
    int64_t lo = 0, hi = nrec - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (rec_base[mid] <= slot) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// prepare: each chunk's entries stably ordered by mode (plain bits, trits,
// quints, undecoded); entry.y = descriptor | channel << 5 | index in chunk << 7
__global__ void __launch_bounds__(THREADS) k_sort_chunks(Ws w, uint64_t ntot) {
    __shared__ int part[4][THREADS + 1];
    const int tid = threadIdx.x;
    const uint64_t c0 = (uint64_t)blockIdx.x * PAY_CHUNK;
    constexpr int EPT = PAY_CHUNK / THREADS;
    uint2 e[EPT];
    int m[EPT];
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const uint64_t i = c0 + tid * EPT + q;
        e[q] = i < ntot ? w.entries[i] : make_uint2(0u, SKIP);
        const uint32_t d = e[q].y & 31u;
        m[q] = d < (uint32_t)NUM_DESC ? desc_mode((int)d) : 3;
    }
    for (int mm = 0; mm < 4; ++mm) {
        int cnt = 0;
#pragma unroll
        for (int q = 0; q < EPT; ++q) cnt += m[q] == mm;
        part[mm][tid + 1] = cnt;
    }
    if (tid == 0)
        for (int mm = 0; mm < 4; ++mm) part[mm][0] = 0;
    __syncthreads();
    if (tid < 4)
        for (int i = 1; i <= THREADS; ++i) part[tid][i] += part[tid][i - 1];
    __syncthreads();
    int base[4];
    base[0] = 0;
    for (int mm = 1; mm < 4; ++mm) base[mm] = base[mm - 1] + part[mm - 1][THREADS];
    int seen[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int mm = m[q];
        const int pos = base[mm] + part[mm][tid] + seen[mm]++;
        const uint32_t local = (uint32_t)(tid * EPT + q);
        w.sorted[c0 + pos] = make_uint2(e[q].x, (e[q].y & 127u) | local << 7);
    }
}

template <int BSQ, typename VT>
__global__ void __launch_bounds__(THREADS) k_payloads(const __grid_constant__ rlfc_field f, Ws w, int l2_last,
                                                      int by_lo, int by_hi, const uint32_t* sel) {
    if (sel && __ldg(sel) <= (uint32_t)SEL_MAX) return;     // k_payloads_sel decoded what the slots need
    __shared__ uint32_t range[2][3];         // per buffer: min / max payload offset, channel mask
    __shared__ uint16_t lut[243 + 125];
    __shared__ VT dq[BSQ == 16 ? 2048 : 1];
    extern __shared__ __align__(16) uint32_t cbuf[];    // [2][PAY_BUF / 4] (B = 4 only)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");      // k_blend's prologue may start
    const int tid = threadIdx.x;
    const int shift = f.quant_shift;
    for (int i = tid; i < 243 + 125; i += THREADS) lut[i] = i < 243 ? g_lut.trit[i] : g_lut.quint[i - 243];
    if (BSQ == 16)
        for (int z = tid; z < 2048; z += THREADS) dq[z] = (VT)deq((uint32_t)z, shift);
    const int64_t nblk = (int64_t)f.wb * f.hb;
    const uint64_t ntot = min((uint64_t)*w.counter, w.cap);
    // the band's payload slots: per channel one contiguous run [lo, hi)
    // (record bases ascend in record order); the chunks covering them
    uint64_t lo[3], hi[3], ch0[3], nch[3];
    for (int c = 0; c < 3; ++c) {
        const int64_t a = (int64_t)c * nblk + (int64_t)by_lo * f.wb, b = (int64_t)c * nblk + (int64_t)by_hi * f.wb;
        lo[c] = min(a < 3 * nblk ? (uint64_t)w.rec_base[a] : ntot, ntot);
        hi[c] = max(lo[c], min(b < 3 * nblk ? (uint64_t)w.rec_base[b] : ntot, ntot));
        ch0[c] = lo[c] / PAY_CHUNK;
        nch[c] = hi[c] > lo[c] ? (hi[c] + PAY_CHUNK - 1) / PAY_CHUNK - ch0[c] : 0;
    }
    const uint64_t n = nch[0] + nch[1] + nch[2];             // chunks to visit (virtual index)
    auto chunk_of = [&](uint64_t v) -> uint64_t {
        return v < nch[0] ? ch0[0] + v : v < nch[0] + nch[1] ? ch0[1] + (v - nch[0]) : ch0[2] + (v - nch[0] - nch[1]);
    };
    VT* res = static_cast<VT*>(w.res);
    uint64_t pol = 0;
    if (l2_last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    constexpr int EPT = PAY_CHUNK / THREADS;                   // entries per thread
    // entry j of chunk cc for this thread (j = tid + q * THREADS); slots
    // outside the band are skipped
    // the raw entries of a chunk are fetched two chunks ahead (fetch), so
    // their latency hides behind a chunk's decode; process filters them
    auto fetch = [&](uint64_t v, uint2* r) {
        const uint64_t cc = chunk_of(v);
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            const uint64_t i = cc * PAY_CHUNK + tid + q * THREADS;
            r[q] = i < ntot ? __ldg(w.sorted + i) : make_uint2(0u, SKIP);
        }
    };
    auto process = [&](uint64_t v, const uint2* r, uint2* e4, uint32_t* sl) {
        const uint64_t cc = chunk_of(v);
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            uint2 e = r[q];
            const uint64_t slot = cc * PAY_CHUNK + ((e.y >> 7) & (PAY_CHUNK - 1));
            const int c = (int)(e.y >> 5) & 3;
            const uint64_t lc = c == 0 ? lo[0] : c == 1 ? lo[1] : lo[2];
            const uint64_t hc = c == 0 ? hi[0] : c == 1 ? hi[1] : hi[2];
            if (slot < lc || slot >= hc) e.y = SKIP;
            e4[q] = e;
            sl[q] = (uint32_t)slot;
        }
    };
    auto reduce_range = [&](const uint2* e4, int q) {
        if (BSQ != 16) return;
        uint32_t rlo = ~0u, rhi = 0u, cm = 0u;
#pragma unroll
        for (int k2 = 0; k2 < EPT; ++k2)
            if ((e4[k2].y & 31u) < (uint32_t)NUM_DESC) {
                rlo = min(rlo, e4[k2].x);
                rhi = max(rhi, e4[k2].x);
                cm |= 1u << ((e4[k2].y >> 5) & 3);
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            rlo = min(rlo, __shfl_xor_sync(0xffffffffu, rlo, o));
            rhi = max(rhi, __shfl_xor_sync(0xffffffffu, rhi, o));
            cm |= __shfl_xor_sync(0xffffffffu, cm, o);
        }
        if ((tid & 31) == 0 && cm) {
            atomicMin(&range[q][0], rlo);
            atomicMax(&range[q][1], rhi);
            atomicOr(&range[q][2], cm);
        }
    };
    // staged (one channel, range fits): copy issue into buffer q; every
    // thread derives the same (staged, lo16) from range[q]
    auto stage_issue = [&](int q, uint32_t& lo16) -> bool {
        if (BSQ != 16 || !range[q][2] || __popc(range[q][2]) != 1) return false;
        const int sc = __ffs(range[q][2]) - 1;
        lo16 = range[q][0] & ~15u;
        if ((uint64_t)range[q][1] + 48 - lo16 > (uint64_t)PAY_BUF) return false;
        const uint64_t end = min((uint64_t)range[q][1] + 48, f.srv_len[sc] + 16);
        const uint8_t* src = f.srv[sc] + lo16;
        const uint32_t dst = smem_u32(cbuf + q * (PAY_BUF / 4));
        const int n16 = (int)((end - lo16) >> 4);
        for (int k2 = tid; k2 < n16; k2 += THREADS)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * k2), "l"(src + 16 * k2)
                         : "memory");
        return true;
    };
    uint64_t v = blockIdx.x;
    uint2 ent[EPT];
    uint32_t sl[EPT];
    bool staged = false;
    uint32_t lo16 = 0;
    if (tid == 0) {
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
            range[b2][0] = ~0u;
            range[b2][1] = 0u;
            range[b2][2] = 0u;
        }
    }
    __syncthreads();
    uint2 rawn[EPT];                                         // chunk v + gridDim.x
    if (v < n) {
        uint2 r0[EPT];
        fetch(v, r0);
        if (v + gridDim.x < n) fetch(v + gridDim.x, rawn);
        process(v, r0, ent, sl);
        reduce_range(ent, 0);
    }
    __syncthreads();
    if (v < n) staged = stage_issue(0, lo16);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int it = 0; v < n; v += gridDim.x, ++it) {
        const int q = it & 1;
        // range[q ^ 1] was reset in the previous iteration (or the prologue)
        // behind at least one barrier: no barrier here
        const bool has_next = v + gridDim.x < n;
        uint2 entn[EPT];
        uint32_t sln[EPT];
        if (has_next) {
            process(v + gridDim.x, rawn, entn, sln);
            if (v + 2 * (uint64_t)gridDim.x < n) fetch(v + 2 * (uint64_t)gridDim.x, rawn);
            reduce_range(entn, q ^ 1);
        }
        __syncthreads();
        uint32_t lo16n = 0;
        bool stagedn = false;
        if (has_next) stagedn = stage_issue(q ^ 1, lo16n);
        if (tid == 0) {
            // range[q] was read by the previous iteration's stage_issue
            // (before the barrier above); the next iteration fills it
            range[q][0] = ~0u;
            range[q][1] = 0u;
            range[q][2] = 0u;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");     // this chunk's copies
        __syncthreads();
        const uint32_t* cb = cbuf + q * (PAY_BUF / 4);
#pragma unroll
        for (int k2 = 0; k2 < EPT; ++k2) {
            const uint2 e = ent[k2];
            const uint32_t d = e.y & 31u;
            if (d >= (uint32_t)NUM_DESC) continue;
            const int m = desc_mode((int)d);
            const uint64_t slot = sl[k2];
            const int c = (int)(e.y >> 5) & 3;
            const uint32_t b = (uint32_t)desc_bits((int)d);
            VT* out = res + slot * BSQ;
            bool bad;
            if constexpr (BSQ == 16) {
                // payload words from the staged chunk, else straight from HBM
                const uint32_t* sw = staged ? cb + ((e.x - lo16) >> 2)
                                            : reinterpret_cast<const uint32_t*>(f.srv[c] + (e.x & ~3u));
                const uint32_t bit0 = (e.x & 3u) * 8u;
                if (m == MODE_BITS) bad = decode16<MODE_BITS, VT>(sw, bit0, b, lut, dq, out, pol);
                else if (m == MODE_TRIT) bad = decode16<MODE_TRIT, VT>(sw, bit0, b, lut, dq, out, pol);
                else bad = decode16<MODE_QUINT, VT>(sw, bit0, b, lut + 243, dq, out, pol);
            } else {
                const uint8_t* p = f.srv[c] + e.x;
                if (m == MODE_BITS) bad = decode_payload<1, 0, BSQ, VT>(p, lut, b, shift, out);
                else if (m == MODE_TRIT) bad = decode_payload<5, 8, BSQ, VT>(p, lut, b, shift, out);
                else bad = decode_payload<3, 7, BSQ, VT>(p, lut + 243, b, shift, out);
            }
            if (bad) w.rec_flag[record_of_slot(w.rec_base, 3 * nblk, slot)] = 1u;   // kernels.py:147-150
        }
        __syncthreads();
#pragma unroll
        for (int k2 = 0; k2 < EPT; ++k2) {
            ent[k2] = entn[k2];
            sl[k2] = sln[k2];
        }
        staged = stagedn;
        lo16 = lo16n;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// ---- pass 2b: slot-mode payloads (small view sets) -------------------------------------
// A decode of a few views (the renderer's tap cameras) needs only the chain
// nodes of those views at levels >= k: for each, one node per record.
// k_sel_nodes collects them (ascending serial index; count first, SEL_MAX + 1
// when there are more); k_payloads_sel then tests each (record, node) pair
// against the prepared bitmap words, and decodes the present ones into their
// slots -- the same residual layout k_payloads writes, so k_blend is unchanged.
__global__ void __launch_bounds__(256) k_sel_nodes(const __grid_constant__ rlfc_field f, const int32_t* slots, int k,
                                                   uint32_t* sel) {
    constexpr int MW = 512;                        // mask words: up to 16384 nodes
    __shared__ uint32_t mask[MW];
    __shared__ uint32_t wcnt[MW + 1];
    const int tid = threadIdx.x;
    if (f.m_nodes > MW * 32) {
        if (tid == 0) sel[0] = SEL_MAX + 1;
        return;
    }
    const int nw = (f.m_nodes + 31) / 32;
    for (int i = tid; i < MW; i += 256) mask[i] = 0u;
    __syncthreads();
    const int T = f.t_count, nv = f.s_count * T;
    for (int v = tid; v < nv; v += 256) {
        if (slots[v] < 0) continue;
        const int s = v / T, t = v - s * T;
        for (int l = k; l < f.tree_height; ++l) {
            const int n = chain_node(f, l, s, t);
            atomicOr(&mask[n >> 5], 1u << (n & 31));
        }
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t run = 0;
        for (int i = 0; i < nw; ++i) {
            wcnt[i] = run;
            run += __popc(mask[i]);
        }
        wcnt[nw] = run;
        sel[0] = run <= (uint32_t)SEL_MAX ? run : (uint32_t)SEL_MAX + 1;
    }
    __syncthreads();
    if (wcnt[nw] > (uint32_t)SEL_MAX) return;
    for (int i = tid; i < nw; i += 256) {
        uint32_t m = mask[i], o = wcnt[i];
        while (m) {
            sel[1 + o++] = (uint32_t)(32 * i + __ffs(m) - 1);
            m &= m - 1u;
        }
    }
}

template <int BSQ, typename VT>
__global__ void __launch_bounds__(THREADS) k_payloads_sel(const __grid_constant__ rlfc_field f, Ws w, int by_lo,
                                                          int by_hi, const uint32_t* __restrict__ sel) {
    constexpr int G8 = 8;                                  // nodes per round
    __shared__ uint16_t lut[243 + 125];
    __shared__ VT dq[BSQ == 16 ? 2048 : 1];
    __shared__ uint32_t nodes[SEL_MAX];
    __shared__ uint2 qe[THREADS * G8];                     // present payloads of the round: entry,
    __shared__ uint32_t qs[THREADS * G8];                  // slot,
    __shared__ uint32_t qr[THREADS * G8];                  // record
    __shared__ int qn;
    const uint32_t cnt = __ldg(sel);
    if (cnt > (uint32_t)SEL_MAX || cnt == 0) return;
    const int tid = threadIdx.x;
    const int shift = f.quant_shift;
    for (int i = tid; i < 243 + 125; i += THREADS) lut[i] = i < 243 ? g_lut.trit[i] : g_lut.quint[i - 243];
    if (BSQ == 16)
        for (int z = tid; z < 2048; z += THREADS) dq[z] = (VT)deq((uint32_t)z, shift);
    for (int i = tid; i < (int)cnt; i += THREADS) nodes[i] = __ldg(sel + 1 + i);
    // one thread per record finds the round's present nodes (bitmap word and
    // slot rank loads issued together); the CTA then decodes the compacted
    // payloads with every lane busy (present nodes are sparse: decoding in
    // place left ~6 active lanes per warp)
    const int64_t nblk = (int64_t)f.wb * f.hb, nrec = 3 * nblk;
    const int64_t nb = (int64_t)(by_hi - by_lo) * f.wb;
    const int64_t r = (int64_t)blockIdx.x * THREADS + tid;
    const bool valid = r < 3 * nb;
    const int c = valid ? (int)(r / nb) : 0;
    const int64_t ri = valid ? (int64_t)c * nblk + (int64_t)by_lo * f.wb + (r - (int64_t)c * nb) : 0;
    const bool live = valid && !__ldg(w.rec_flag + ri);       // anomalous records: k_fixup
    VT* res = static_cast<VT*>(w.res);
    for (int j0 = 0; j0 < (int)cnt; j0 += G8) {
        if (tid == 0) qn = 0;
        __syncthreads();
        if (live) {
            uint32_t word[G8], rk[G8];
#pragma unroll
            for (int q = 0; q < G8; ++q) {
                word[q] = 0u;
                rk[q] = 0u;
                if (j0 + q < (int)cnt) {
                    const int64_t o = (int64_t)(nodes[j0 + q] >> 5) * nrec + ri;
                    word[q] = __ldg(w.bm + o);
                    rk[q] = __ldg(w.rk + o);
                }
            }
#pragma unroll
            for (int q = 0; q < G8; ++q) {
                const uint32_t n = j0 + q < (int)cnt ? nodes[j0 + q] : 0u;
                if (j0 + q < (int)cnt && ((word[q] >> (n & 31u)) & 1u)) {
                    const uint32_t slot = rk[q] + (uint32_t)__popc(word[q] & ((1u << (n & 31u)) - 1u));
                    if (slot < w.cap) {
                        const int pos = atomicAdd(&qn, 1);
                        qe[pos] = __ldg(w.entries + slot);
                        qs[pos] = slot;
                        qr[pos] = (uint32_t)ri;
                    }
                }
            }
        }
        __syncthreads();
        const int n = qn;
        for (int i = tid; i < n; i += THREADS) {
            const uint2 e = qe[i];
            const uint32_t d = e.y & 31u;
            if (d >= (uint32_t)NUM_DESC) continue;
            const int m = desc_mode((int)d);
            const int cc = (int)(e.y >> 5) & 3;
            const uint32_t b = (uint32_t)desc_bits((int)d);
            VT* out = res + (uint64_t)qs[i] * BSQ;
            bool bad;
            if constexpr (BSQ == 16) {
                const uint32_t* sw = reinterpret_cast<const uint32_t*>(f.srv[cc] + (e.x & ~3u));
                const uint32_t bit0 = (e.x & 3u) * 8u;
                if (m == MODE_BITS) bad = decode16<MODE_BITS, VT>(sw, bit0, b, lut, dq, out);
                else if (m == MODE_TRIT) bad = decode16<MODE_TRIT, VT>(sw, bit0, b, lut, dq, out);
                else bad = decode16<MODE_QUINT, VT>(sw, bit0, b, lut + 243, dq, out);
            } else {
                const uint8_t* p = f.srv[cc] + e.x;
                if (m == MODE_BITS) bad = decode_payload<1, 0, BSQ, VT>(p, lut, b, shift, out);
                else if (m == MODE_TRIT) bad = decode_payload<5, 8, BSQ, VT>(p, lut, b, shift, out);
                else bad = decode_payload<3, 7, BSQ, VT>(p, lut + 243, b, shift, out);
            }
            if (bad) w.rec_flag[qr[i]] = 1u;                     // kernels.py:147-150
        }
        __syncthreads();
    }
}

// ---- pass 3: blend -------------------------------------------------------------------
#ifdef RLFC_BLEND_TIMING
// per-CTA %globaltimer stamps of k_blend (debug build, tools/blend_timing.py):
// start, records done, sync1, units done, TMA wait + sync2, tasks done, sync3,
// store read
__device__ long long g_btime[65536 * 8];
#define RLFC_BSTAMP(q) do { if (threadIdx.x == 0 && bidx < 65536) { long long tt; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt)); g_btime[bidx * 8 + (q)] = tt; } } while (0)
#else
#define RLFC_BSTAMP(q) do { } while (0)
#endif

struct BlendParams {
    rlfc_field f;
    int k;
    const int32_t* slots;
    int by_lo;
    uint8_t* rgb;
    int64_t img_stride, row_stride;
    uint64_t* status;
    const uint32_t* rec_base;
    const uint32_t* rec_flag;
    const void* res;
    const uint8_t* root_rgb_g;   // RGB8 of every root sample [root][hp][rgb_stride]
    int rgb_stride;
    const uint32_t* bm;          // record bitmap words / word ranks (k_index)
    const uint32_t* rk;
    int nwp;
    int TW, NB, nchunks, nstrip;
    int store_mode;              // 2: TMA tensor stores, 1: per-row bulk copies, 0: byte stores
    int store_keep;              // 1: output stores with the normal L2 policy, 0: evict-first
    int tma_in;                  // 1: staging and raw roots arrive by TMA tensor loads
    int roots_vec;               // root rows are 16-byte aligned in HBM (manual path)
    const int32_t* trows;        // camera rows to decode (grid.y indexes it), or null = all
    uint32_t* units;             // prepared dirty-unit lists (B = 4), or null
    int ucap;
    int build_units;             // 1: this launch writes the lists (prepare, k = 0)
    int off_flag, off_mask, off_sbase, off_roots, off_rgb, off_cnt, off_list, off_stage,
        off_mbar;
};

__device__ __forceinline__ uint32_t pack4_sat(int32_t b0, int32_t b1, int32_t b2, int32_t b3) {
    uint32_t hi, d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(hi) : "r"(b3), "r"(b2), "r"(0));
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(b1), "r"(b0), "r"(hi));
    return d;
}

// colorspace.py:27-36 on four pixels, packed to 12 RGB bytes.
__device__ __forceinline__ void ycocg4_pack(const int32_t (*v)[4], uint32_t* o3) {
    int32_t o[12];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int32_t tt = v[0][i] - (v[2][i] >> 1);
        const int32_t bb = tt - (v[1][i] >> 1);
        o[3 * i] = bb + v[1][i];
        o[3 * i + 1] = v[2][i] + tt;
        o[3 * i + 2] = bb;
    }
    o3[0] = pack4_sat(o[0], o[1], o[2], o[3]);
    o3[1] = pack4_sat(o[4], o[5], o[6], o[7]);
    o3[2] = pack4_sat(o[8], o[9], o[10], o[11]);
}

template <typename RT>
__device__ __forceinline__ void load4s(const RT* p, int32_t* v) {
    if (sizeof(RT) == 2) {
        const uint2 w = *reinterpret_cast<const uint2*>(p);
        v[0] = (int32_t)(int16_t)(w.x & 0xFFFFu);
        v[1] = (int32_t)w.x >> 16;
        v[2] = (int32_t)(int16_t)(w.y & 0xFFFFu);
        v[3] = (int32_t)w.y >> 16;
    } else {
        const int4 w = *reinterpret_cast<const int4*>(p);
        v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
    }
}

// ---- root colours: RGB8 of every root sample (colorspace.py:27-56) -------------------
template <typename RT>
__global__ void __launch_bounds__(THREADS) k_root_rgb(const __grid_constant__ rlfc_field f, uint8_t* out,
                                                      int rgb_stride, int y0, int y1) {
    const int quads = f.wp / 4;
    const int rows = y1 - y0;
    const int64_t n = (int64_t)f.rsx * f.rsy * rows * quads;
    const int64_t pl = (int64_t)f.hp * f.wp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int xq = (int)(i % quads);
        const int64_t rr = i / quads;                  // root * rows + (y - y0)
        const int y = y0 + (int)(rr % rows);
        const int64_t r = rr / rows;
        const int64_t ry = r * f.hp + y;
        int32_t v[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const RT* src = reinterpret_cast<const RT*>(f.roots) + (r * 3 + c) * pl + (int64_t)y * f.wp + xq * 4;
#pragma unroll
            for (int j = 0; j < 4; ++j) v[c][j] = (int32_t)src[j];
        }
        ycocg4_pack(v, reinterpret_cast<uint32_t*>(out + ry * rgb_stride + xq * 12));
    }
    // launched programmatically behind k_index: do not complete before it
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// byte offset of pixel (view s, row, tile column px) in the strip-major
// staging buffer [strip][S][B][STRIP*3]
template <int B>
__device__ __forceinline__ int stage_off(int S, int s, int row, int px) {
    return (((px / STRIP) * S + s) * B + row) * (STRIP * 3) + (px % STRIP) * 3;
}

// (view, block) units touching a record with a stream anomaly (bad
// descriptor, truncation, corrupt pack: listed by rlfc_staged_prepare) are
// skipped by the blend and redone afterwards by the reference-order walk
// (kernels.py:162-216, decode_chain_core) for all three channels, over the
// blend's output, with the failure word keyed as the reference meets it.
template <int B>
__global__ void k_fixup(const __grid_constant__ rlfc_field f, const uint32_t* flist, int k, const int32_t* slots,
                        int by_lo, int by_hi, uint8_t* rgb, int64_t img_stride, int64_t row_stride,
                        uint64_t* status) {
    constexpr int BSQ = B * B;
    const int64_t nblk = (int64_t)f.wb * f.hb;
    const int64_t ri = flist[1 + blockIdx.x];
    const int64_t blk = ri % nblk;
    const int by = (int)(blk / f.wb), bx = (int)(blk % f.wb);
    if (by < by_lo || by >= by_hi) return;
    const int v = blockIdx.y * blockDim.x + threadIdx.x;
    if (v >= f.s_count * f.t_count) return;
    const int slot = slots ? slots[v] : v;
    if (slot < 0) return;
    const int s = v / f.t_count, t = v % f.t_count;
    int32_t acc[3][BSQ];
    for (int c = 0; c < 3; ++c) {
        for (int yy = 0; yy < B; ++yy)
            for (int xx = 0; xx < B; ++xx) acc[c][yy * B + xx] = root_sample(f, s, t, c, by * B + yy, bx * B + xx);
        const uint64_t off = f.offsets[c][blk];
        int st = walk_chain<BSQ>(f, f.srv[c] + off, s, t, k, acc[c], g_lut, node_bytes<BSQ>(), srv_avail(f, c, off));
        if (st == WALK_OOB) st = 2;
        if (st) {
            report(status, ((((uint64_t)v) * 3 + c) * f.hb + by) * f.wb + bx, st);
            return;
        }
    }
    for (int yy = 0; yy < B; ++yy) {
        const int y = by * B + yy;
        if (y >= f.height) break;
        uint8_t* orow = rgb + (int64_t)slot * img_stride + (int64_t)(y - by_lo * B) * row_stride;
        for (int xx = 0; xx < B; ++xx) {
            const int x = bx * B + xx;
            if (x >= f.width) break;
            uint32_t r, g, b;
            ycocg_to_rgb8(acc[0][yy * B + xx], acc[1][yy * B + xx], acc[2][yy * B + xx], r, g, b);
            orow[3 * x] = (uint8_t)r;
            orow[3 * x + 1] = (uint8_t)g;
            orow[3 * x + 2] = (uint8_t)b;
        }
    }
}

// Random-access block decode over the prepared record index (decoder.py:
// 81-106 / kernels.py:162-216): per chain level, the node's presence bit and
// payload slot come from the record's bitmap word and word rank (one round
// trip for all levels), the slot's entry gives the payload's byte offset
// and descriptor, and only the chain payloads are read and BISE-decoded -- no
// walk over the record's earlier nodes.  Records with a stream anomaly take
// the reference-order walk.  Out-of-range requests report code 3.
// One BISE mode's payloads of a lane's chain (levels in pm) added into acc,
// one per round; the entry of the round's level is picked by predicated
// selects (no dynamic register indexing).
template <int MODE>
__device__ __forceinline__ bool indexed_mode_rounds(const rlfc_field& f, int c, const uint2 (&ent)[MAXH], uint32_t pm,
                                                    int32_t* acc) {
    bool bad = false;
    while (pm) {
        const int l = __ffs(pm) - 1;
        pm &= pm - 1u;
        uint2 e = make_uint2(0u, 0u);
#pragma unroll
        for (int ll = 0; ll < MAXH; ++ll)
            if (ll == l) e = ent[ll];
        const uintptr_t a = reinterpret_cast<uintptr_t>(f.srv[c] + e.x);
        const uint32_t* sw = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
        const uint32_t bit0 = (uint32_t)(a & 3u) * 8u, b = (uint32_t)desc_bits((int)(e.y & 31u));
        bad |= decode16_acc<MODE>(sw, bit0, b,
                                  MODE == MODE_BITS ? nullptr : MODE == MODE_TRIT ? g_lut.trit : g_lut.quint,
                                  f.quant_shift, acc);
    }
    return bad;
}

template <int B>
__global__ void k_blocks_indexed(const __grid_constant__ rlfc_field f, Ws w, const int32_t* __restrict__ req, int n,
                                 int32_t* __restrict__ out, int32_t* __restrict__ status) {
    constexpr int BSQ = B * B;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = req[6 * i], t = req[6 * i + 1], bx = req[6 * i + 2], by = req[6 * i + 3];
    int c = req[6 * i + 4];
    const int k = req[6 * i + 5];
    if (s < 0 || s >= f.s_count || t < 0 || t >= f.t_count || bx < 0 || bx >= f.wb || by < 0 || by >= f.hb ||
        c < -3 || c >= 3 || k < 0 || k > f.tree_height) {
        status[i] = 3;
        return;
    }
    if (c < 0) c += 3;
    const int64_t nblk = (int64_t)f.wb * f.hb, nrec = 3 * nblk;
    const int64_t blk = (int64_t)by * f.wb + bx, ri = (int64_t)c * nblk + blk;
    int32_t acc[BSQ];
    if (B == 4 && f.roots_i16) {
        // the block's four root rows: one aligned 8-byte load each
        const int h = f.tree_height;
        const int16_t* r0 = reinterpret_cast<const int16_t*>(f.roots) +
                            ((((int64_t)(s >> h) * f.rsy + (t >> h)) * 3 + c) * f.hp + by * B) * f.wp + bx * B;
#pragma unroll
        for (int yy = 0; yy < B; ++yy) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(r0 + (int64_t)yy * f.wp));
            acc[yy * B] = (int32_t)(int16_t)(v.x & 0xFFFFu);
            acc[yy * B + 1] = (int32_t)v.x >> 16;
            acc[yy * B + 2] = (int32_t)(int16_t)(v.y & 0xFFFFu);
            acc[yy * B + 3] = (int32_t)v.y >> 16;
        }
    } else {
#pragma unroll
        for (int yy = 0; yy < B; ++yy)
#pragma unroll
            for (int xx = 0; xx < B; ++xx) acc[yy * B + xx] = root_sample(f, s, t, c, by * B + yy, bx * B + xx);
    }
    int st = 0;
    if (__ldg(w.rec_flag + ri)) {
        const uint64_t off = f.offsets[c][blk];
        st = walk_chain<BSQ>(f, f.srv[c] + off, s, t, k, acc, g_lut, node_bytes<BSQ>(), srv_avail(f, c, off));
        if (st == WALK_OOB) st = 2;
    } else {
        const int h = f.tree_height;
        uint32_t words[MAXH], ranks[MAXH];
#pragma unroll
        for (int l = 0; l < MAXH; ++l) {
            words[l] = ranks[l] = 0u;
            if (l >= k && l < h) {
                const int nd = chain_node(f, l, s, t);
                words[l] = __ldg(w.bm + (int64_t)(nd >> 5) * nrec + ri);
                ranks[l] = __ldg(w.rk + (int64_t)(nd >> 5) * nrec + ri);
            }
        }
        uint2 ent[MAXH];
#pragma unroll
        for (int l = 0; l < MAXH; ++l) {
            ent[l] = make_uint2(0u, SKIP);
            if (l >= k && l < h) {
                const int bit = chain_node(f, l, s, t) & 31;
                if ((words[l] >> bit) & 1u)
                    ent[l] = __ldg(w.entries + ranks[l] + __popc(words[l] & ((1u << bit) - 1u)));
            }
        }
        if constexpr (BSQ == 16) {
            // mode-major: a lane decodes its present levels one BISE mode at
            // a time, so each round of a warp runs one mode's code for every
            // lane that has a payload of that mode (level-major rounds ran a
            // body per (level, mode) pair present anywhere in the warp). The
            // level sums are integer additions, so their order is free; an
            // unflagged record has no corrupt pack (prepare validated it).
            uint32_t pm[3] = {0u, 0u, 0u};
#pragma unroll
            for (int l = 0; l < MAXH; ++l) {
                const uint32_t d = ent[l].y & 31u;
                if (d < (uint32_t)NUM_DESC) {
                    const int m = desc_mode((int)d);
                    pm[0] |= (m == MODE_BITS ? 1u : 0u) << l;
                    pm[1] |= (m == MODE_TRIT ? 1u : 0u) << l;
                    pm[2] |= (m == MODE_QUINT ? 1u : 0u) << l;
                }
            }
            bool bad = false;
            bad |= indexed_mode_rounds<MODE_BITS>(f, c, ent, pm[0], acc);
            bad |= indexed_mode_rounds<MODE_TRIT>(f, c, ent, pm[1], acc);
            bad |= indexed_mode_rounds<MODE_QUINT>(f, c, ent, pm[2], acc);
            st = bad ? 1 : 0;
        } else {
            // chain order h-1 .. k, as the reference decodes its targets
#pragma unroll
            for (int l = MAXH - 1; l >= 0; --l) {
                const uint32_t d = ent[l].y & 31u;
                if (d >= (uint32_t)NUM_DESC || st) continue;
                st = decode_payload_acc<BSQ>(f.srv[c] + ent[l].x, (int)d, f.quant_shift, acc, g_lut);
            }
        }
    }
    status[i] = st;
    int32_t* o = out + (int64_t)i * BSQ;
    if constexpr (BSQ % 4 == 0) {
#pragma unroll
        for (int j = 0; j < BSQ; j += 4)
            *reinterpret_cast<int4*>(o + j) = make_int4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < BSQ; ++j) o[j] = acc[j];
    }
}

__global__ void k_flag_list(const uint32_t* rec_flag, int64_t nrec, uint32_t* flist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nrec && rec_flag[i]) flist[1 + atomicAdd(flist, 1u)] = (uint32_t)i;
}

// NL: present chain levels per unit held in registers (1; RLFC_DENSE_NL for
// dense streams, whose units often carry several present levels, at fewer
// CTAs per SM); further levels are read row by row.
template <int B, typename VT, typename RT, int BT, int NL = 1>
#ifndef RLFC_BLEND_MINB
#define RLFC_BLEND_MINB (1024 / BT)
#endif
// dense variant: two levels in registers at 8 CTAs per SM measured best
// (cfg2 R6: 1.40 ms vs 1.84 ms one level, 1.45 ms three levels at 6 CTAs;
// R5: 0.94 vs 1.09 ms; R4 is faster with one level: 0.438 vs 0.488 ms)
#ifndef RLFC_DENSE_MINB
#define RLFC_DENSE_MINB 8
#endif
#ifndef RLFC_DENSE_NL
#define RLFC_DENSE_NL 2
#endif
__global__ void __launch_bounds__(BT, NL == 1 ? RLFC_BLEND_MINB : RLFC_DENSE_MINB) k_blend(const __grid_constant__ BlendParams P,
                                                   const __grid_constant__ CUtensorMap out_map,
                                                   const __grid_constant__ CUtensorMap rgb_map,
                                                   const __grid_constant__ CUtensorMap root_map) {
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int BSQ = B * B;
    constexpr int QB = B / 4;                      // pixel quads per block row
    const rlfc_field& f = P.f;
    const int tid = threadIdx.x;
    const int chunk = blockIdx.x, t = P.trows ? P.trows[blockIdx.y] : (int)blockIdx.y;
    const int by = P.by_lo + blockIdx.z;
    const int NB = P.NB, TW = P.TW, NR = 3 * NB;
    const int bx0 = chunk * NB;
    const int nb = min(NB, f.wb - bx0);
    const int h = f.tree_height, k = P.k, S = f.s_count, T = f.t_count;
    const int nlev = h - k;
    const int ry = t >> h;
    const int64_t nblk = (int64_t)f.wb * f.hb;

    uint32_t* rflag = reinterpret_cast<uint32_t*>(smem + P.off_flag);       // [NR]
    uint64_t* mask = reinterpret_cast<uint64_t*>(smem + P.off_mask);        // [nlev][NR]
    uint32_t* sbase = reinterpret_cast<uint32_t*>(smem + P.off_sbase);      // [nlev][NR]
    RT* roots = reinterpret_cast<RT*>(smem + P.off_roots);                 // [rsx][3][B][TW]
    uint8_t* root_rgb = smem + P.off_rgb;                                   // [strip][rsx][B][STRIP*3] (manual)
    int32_t* cnt = reinterpret_cast<int32_t*>(smem + P.off_cnt);            // [0] units, [1] warp-0 total
    uint2* list = reinterpret_cast<uint2*>(smem + P.off_list);              // [S*NB]
    uint8_t* stage = smem + P.off_stage;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + P.off_mbar);
#ifdef RLFC_BLEND_TIMING
    const int64_t bidx = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#endif
    RLFC_BSTAMP(0);

    // ---- TMA: RGB(root) rows into every view's staging rows, raw roots ----------------
    if (P.tma_in && tid >= BT - 32) {
        // last warp (no record work when NR <= BT - 32): lane 0 arms the
        // barrier, then every lane issues its share of the tensor loads
        const uint32_t bar = smem_u32(mbar);
        // with a slot table only the requested views of this camera row are
        // prefilled (their count sets the barrier's byte count)
        const int ln = tid - (BT - 32);
        uint32_t need = 0;
        for (int s0 = 0; s0 < S; s0 += 32) {
            const int s = s0 + ln;
            const bool want = s < S && (!P.slots || P.slots[s * T + t] >= 0);
            need += __popc(__ballot_sync(0xffffffffu, want));
        }
        if (tid == BT - 32) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const uint32_t bytes =
                (uint32_t)(P.nstrip * need * B * STRIP * 3) + (uint32_t)(f.rsx * 3 * B * TW * (int)sizeof(RT));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        }
        __syncwarp();
        const int nrgb = P.nstrip * S;
        for (int i = tid - (BT - 32); i < nrgb + f.rsx * 3; i += 32) {
            if (i < nrgb) {
                const int st = i / S, s = i - st * S;
                if (P.slots && P.slots[s * T + t] < 0) continue;
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                    "%4}], [%5];" ::"r"(smem_u32(stage + ((st * S + s) * B) * (STRIP * 3))),
                    "l"(&rgb_map), "r"((bx0 * B + st * STRIP) * 3), "r"(by * B), "r"((s >> h) * f.rsy + ry), "r"(bar)
                    : "memory");
            } else {
                const int q = i - nrgb, rx = q / 3, c = q - rx * 3;
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                    "%4}], [%5];" ::"r"(smem_u32(roots + (rx * 3 + c) * B * TW)),
                    "l"(&root_map), "r"(bx0 * B), "r"(by * B), "r"((rx * f.rsy + ry) * 3 + c), "r"(bar)
                    : "memory");
            }
        }
    }

    if (tid == 0) cnt[0] = 0;
    // prepared dirty-unit list of this tile (B = 4): its count and this
    // thread's first two entries are loaded with the record tables (one round
    // trip); the pair scan below is then skipped
    const bool use_list = B == 4 && P.units && !P.build_units;
    const uint32_t* ulist = nullptr;
    uint32_t ucount = 0, ue0 = 0, ue1 = 0;
    if (use_list) {
        ulist = P.units + ((uint64_t)((int64_t)by * T + t) * P.nchunks + chunk) * (uint64_t)(1 + P.ucap);
        ucount = __ldg(ulist);
        if (tid < P.ucap) ue0 = __ldg(ulist + 1 + tid);
        if (tid + BT < P.ucap) ue1 = __ldg(ulist + 1 + tid + BT);
    }
    // ---- records: residual row masks and slot bases of this camera row --------
    for (int r = tid; r < NR; r += BT) {
        const int c = r >> (__ffs(NB) - 1), b = r & (NB - 1);
        uint32_t fl = 0;
        if (b < nb && nlev > 0) {
            const int64_t blk = (int64_t)by * f.wb + bx0 + b;
            const int64_t ri = (int64_t)c * nblk + blk;
            {
                // every table word of the first RL levels is loaded before
                // any is used (one round trip, not one per level); they are
                // loaded regardless of the flag (stale for flagged records,
                // which never read them)
                constexpr int RL = 3;
                const int64_t nrec = 3 * nblk;
                const uint32_t* bmr = P.bm + ri;
                const uint32_t* rkr = P.rk + ri;
                uint32_t lo[RL], hi[RL], hi2[RL], rkv[RL];
#pragma unroll
                for (int li = 0; li < RL; ++li) {
                    lo[li] = hi[li] = hi2[li] = rkv[li] = 0u;
                    if (li < nlev) {
                        const int l = k + li, sx = f.level_sx[l];
                        const int wi = (f.level_base[l] + (t >> l) * sx) >> 5;
                        lo[li] = __ldg(bmr + wi * nrec);
                        hi[li] = __ldg(bmr + (wi + 1) * nrec);
                        if (sx > 32) hi2[li] = __ldg(bmr + (wi + 2) * nrec);
                        rkv[li] = __ldg(rkr + wi * nrec);
                    }
                }
                // the table words above come from k_index (complete); the flags
                // are also written by k_payloads, which may still be running
                // when this grid starts (programmatic launch). The flag load is
                // issued before any table word is consumed, so both share one
                // round trip. A coherent load the compiler cannot hoist above
                // the wait (ld.global.nc may be scheduled early).
                asm volatile("griddepcontrol.wait;" ::: "memory");
                asm volatile("ld.global.u32 %0, [%1];" : "=r"(fl) : "l"(P.rec_flag + ri) : "memory");
#pragma unroll
                for (int li = 0; li < RL; ++li) {
                    if (li < nlev) {
                        const int l = k + li, sx = f.level_sx[l];
                        const int o = (f.level_base[l] + (t >> l) * sx) & 31;
                        uint64_t m = __funnelshift_r(lo[li], hi[li], o);
                        if (sx > 32) m |= (uint64_t)__funnelshift_r(hi[li], hi2[li], o) << 32;
                        if (sx < 64) m &= (1ull << sx) - 1ull;
                        mask[li * NR + r] = m;
                        sbase[li * NR + r] = rkv[li] + __popc(lo[li] & ((1u << o) - 1u));
                    }
                }
                for (int li = RL; li < nlev; ++li) {             // deeper trees
                    const int l = k + li, sx = f.level_sx[l];
                    const int n0 = f.level_base[l] + (t >> l) * sx;
                    const int wi = n0 >> 5, o = n0 & 31;
                    const uint32_t a = __ldg(bmr + wi * nrec), c2 = __ldg(bmr + (wi + 1) * nrec);
                    uint64_t m = __funnelshift_r(a, c2, o);
                    if (sx > 32) m |= (uint64_t)__funnelshift_r(c2, __ldg(bmr + (wi + 2) * nrec), o) << 32;
                    if (sx < 64) m &= (1ull << sx) - 1ull;
                    mask[li * NR + r] = m;
                    sbase[li * NR + r] = __ldg(rkr + wi * nrec) + __popc(a & ((1u << o) - 1u));
                }
            }
        } else if (nlev > 0) {
            for (int l = k; l < h; ++l) mask[(l - k) * NR + r] = 0;
        }
        rflag[r] = fl;
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");       // residuals (tasks) come from k_payloads
    // ---- manual path: roots of this camera row and their RGB8 -------------------------
    if (!P.tma_in && !P.build_units) {
        const int quads = TW / 4;
        const int64_t pl = (int64_t)f.hp * f.wp;
        for (int it = tid; it < f.rsx * B * quads; it += BT) {
            const int xq = it % quads, rr = (it / quads) % B, rx = it / (quads * B);
            const int gx = bx0 * B + xq * 4;
            int32_t v[3][4];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const RT* src = reinterpret_cast<const RT*>(f.roots) + (((int64_t)rx * f.rsy + ry) * 3 + c) * pl +
                                (int64_t)(by * B + rr) * f.wp + gx;
                if (P.roots_vec && gx + 4 <= f.wp) {
                    load4s<RT>(src, v[c]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[c][j] = gx + j < f.wp ? (int32_t)src[j] : 0;
                }
                RT* dst = roots + ((rx * 3 + c) * B + rr) * TW + xq * 4;
#pragma unroll
                for (int j = 0; j < 4; ++j) dst[j] = (RT)v[c][j];
            }
            const int px = xq * 4;
            uint32_t* o = reinterpret_cast<uint32_t*>(root_rgb + (((px / STRIP) * f.rsx + rx) * B + rr) * (STRIP * 3) +
                                                      (px % STRIP) * 3);
            ycocg4_pack(v, o);
        }
    }
    RLFC_BSTAMP(1);
    __syncthreads();
    RLFC_BSTAMP(2);

    // ---- dirty (view, block) units: one thread per pair tests the chain's
    // presence bits (bit 3(l-k)+c: level l, channel c) and appends dirty pairs
    // with a warp-aggregated shared-memory atomic (unit order is irrelevant);
    // pairs touching a flagged record are tagged for the reference-order walk
    const int lane = tid & 31;
    const int lgnb = __ffs(NB) - 1;                  // NB is a power of two (TW / B)
    for (int p0 = use_list ? S * NB : 0; p0 < S * NB; p0 += BT) {
        const int pi = p0 + tid;
        const int s = pi >> lgnb, b = pi & (NB - 1);
        bool emit = false, fb = false;
        uint32_t pres = 0;
        if (pi < S * NB && b < nb && (!P.slots || P.slots[s * T + t] >= 0)) {
            fb = (rflag[b] | rflag[NB + b] | rflag[2 * NB + b]) != 0;
            if (!fb) {
                const uint64_t* mb = mask + b;
                for (int li = 0; li < nlev; ++li, mb += NR) {
                    const int x = s >> (k + li);
                    pres |= (uint32_t)((mb[0] >> x) & 1ull) << (3 * li) |
                            (uint32_t)((mb[NB] >> x) & 1ull) << (3 * li + 1) |
                            (uint32_t)((mb[2 * NB] >> x) & 1ull) << (3 * li + 2);
                }
            }
            emit = fb || pres != 0;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, emit);
        if (bal) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&cnt[0], __popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (emit)
                list[base + __popc(bal & ((1u << lane) - 1u))] =
                    make_uint2((uint32_t)s | (uint32_t)b << 8 | (fb ? 1u << 16 : 0u), pres);
        }
    }
    if (P.build_units) {
        // prepare (k = 0): this tile's dirty units (s | b << 8 | presence << 14)
        __syncthreads();
        uint32_t* ul = P.units + ((uint64_t)((int64_t)by * T + t) * P.nchunks + chunk) * (uint64_t)(1 + P.ucap);
        const int n = cnt[0];
        if (tid == 0) ul[0] = (uint32_t)n;
        for (int u = tid; u < n; u += BT) ul[1 + u] = list[u].x & 0xFFFFu | list[u].y << 14;
        return;
    }
    if (!P.tma_in) {
        // staging[strip][s][row] <- root_rgb[strip][s >> h][row]: one warp per
        // staged (strip, view), B*12 16-byte copies
        constexpr int V = B * STRIP * 3 / 16;
        for (int sv = tid >> 5; sv < P.nstrip * S; sv += BT / 32) {
            const int st = sv / S, s = sv - st * S;
            const uint4* src = reinterpret_cast<const uint4*>(root_rgb + (st * f.rsx + (s >> h)) * B * (STRIP * 3));
            uint4* dst = reinterpret_cast<uint4*>(stage + sv * B * (STRIP * 3));
            for (int v = lane; v < V; v += 32) dst[v] = src[v];
        }
    }
    RLFC_BSTAMP(3);
    if (P.tma_in) {
        const uint32_t bar = smem_u32(mbar);
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(bar)
                : "memory");
    }
    __syncthreads();
    RLFC_BSTAMP(4);

    // ---- dirty units: root + present residuals, YCoCg-R inverse, clamp, pack ----------
    // one task = two consecutive pixel quad-rows of a unit (8 consecutive
    // values of each payload), so a present residual is one 16-byte gather
    if constexpr (B == 4 && sizeof(VT) == 2) {
        // B = 4: one task per unit (all 16 pixels): the first present level
        // of each channel is two 16-byte gathers, all issued before any is
        // consumed, so a thread pays one round trip per unit
        const int units = use_list ? (int)ucount : cnt[0];
        const VT* res = static_cast<const VT*>(P.res);
        for (int u = tid; u < units; u += BT) {
            uint2 e;
            if (use_list) {
                // prepared entry (k = 0): keep levels >= k, skip views outside
                // the slot table, units of anomalous records (k_fixup) and
                // units clean at this stop level
                const uint32_t q = u == tid ? ue0 : u == tid + BT ? ue1 : __ldg(ulist + 1 + u);
                const int s = (int)(q & 255u), b = (int)((q >> 8) & 63u);
                const uint32_t pres = (q >> 14 >> (3 * k)) & ((1u << (3 * nlev)) - 1u);
                if (rflag[b] | rflag[NB + b] | rflag[2 * NB + b]) continue;
                if (!pres || (P.slots && P.slots[s * T + t] < 0)) continue;
                e = make_uint2((uint32_t)s | (uint32_t)b << 8, pres);
            } else {
                e = list[u];
            }
            const int s = (int)(e.x & 255u), b = (int)((e.x >> 8) & 255u);
            if (e.x >> 16) continue;                 // anomalous record: k_fixup
            auto slot_of = [&](int c, uint32_t pc) -> uint32_t {
                const int li = (__ffs(pc) - 1) / 3;
                const int r = li * NR + c * NB + b;
                const int x = s >> (k + li);
                return sbase[r] + (uint32_t)__popcll(mask[r] & ((1ull << x) - 1ull));
            };
            uint4 raw[NL][3][2];
            uint32_t pcs[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                pcs[c] = e.y & (0x249249u << c);             // bits 3i + c: levels k + i
#pragma unroll
                for (int lv = 0; lv < NL; ++lv) {
                    raw[lv][c][0] = raw[lv][c][1] = make_uint4(0u, 0u, 0u, 0u);
                    if (pcs[c]) {
                        // the payload's 32-byte sector in one 256-bit load
                        const VT* q = res + (uint64_t)slot_of(c, pcs[c]) * BSQ;
                        asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                            : "=r"(raw[lv][c][0].x), "=r"(raw[lv][c][0].y), "=r"(raw[lv][c][0].z),
                              "=r"(raw[lv][c][0].w), "=r"(raw[lv][c][1].x), "=r"(raw[lv][c][1].y),
                              "=r"(raw[lv][c][1].z), "=r"(raw[lv][c][1].w)
                            : "l"(q));
                        pcs[c] &= pcs[c] - 1u;
                    }
                }
            }
            const int rx = s >> h;
            const int px = b * B;
#pragma unroll
            for (int row = 0; row < 4; ++row) {
                int32_t v[3][4];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    load4s<RT>(roots + ((rx * 3 + c) * B + row) * TW + px, v[c]);
#pragma unroll
                    for (int lv = 0; lv < NL; ++lv) {
                        const uint4 w = raw[lv][c][row >> 1];
                        const uint32_t lo = (row & 1) ? w.z : w.x, hi = (row & 1) ? w.w : w.y;
                        v[c][0] += (int32_t)(int16_t)(lo & 0xFFFFu);
                        v[c][1] += (int32_t)lo >> 16;
                        v[c][2] += (int32_t)(int16_t)(hi & 0xFFFFu);
                        v[c][3] += (int32_t)hi >> 16;
                    }
                    uint32_t pc = pcs[c];
                    while (pc) {                               // further levels (rare)
                        int32_t r4[4] = {0, 0, 0, 0};
                        const VT* q = res + (uint64_t)slot_of(c, pc) * BSQ + row * 4;
                        add4<VT>(q, r4);
#pragma unroll
                        for (int i = 0; i < 4; ++i) v[c][i] += r4[i];
                        pc &= pc - 1u;
                    }
                }
                ycocg4_pack(v, reinterpret_cast<uint32_t*>(stage + stage_off<B>(S, s, row, px)));
            }
        }
    } else {
        constexpr int TP = B * QB / 2;                   // tasks per unit
        const int units = use_list ? (int)ucount : cnt[0];
        const VT* res = static_cast<const VT*>(P.res);
        for (int it = tid; it < units * TP; it += BT) {
            const int u = it / TP, j = it - u * TP;
            uint2 e;
            if (use_list) {
                // prepared entry (B = 4, 32-bit residuals): filtered as above
                const uint32_t q = __ldg(ulist + 1 + u);
                const int s = (int)(q & 255u), b = (int)((q >> 8) & 63u);
                const uint32_t pres = (q >> 14 >> (3 * k)) & ((1u << (3 * nlev)) - 1u);
                if (rflag[b] | rflag[NB + b] | rflag[2 * NB + b]) continue;
                if (!pres || (P.slots && P.slots[s * T + t] < 0)) continue;
                e = make_uint2((uint32_t)s | (uint32_t)b << 8, pres);
            } else {
                e = list[u];
            }
            const int s = (int)(e.x & 255u), b = (int)((e.x >> 8) & 255u);
            if (e.x >> 16) continue;                 // anomalous record: k_fixup
            const int rx = s >> h;
            int row[2], px[2];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int qi = 2 * j + hh;
                row[hh] = qi / QB;
                px[hh] = b * B + (qi - row[hh] * QB) * 4;
            }
            int32_t v[2][3][4];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int c = 0; c < 3; ++c) load4s<RT>(roots + ((rx * 3 + c) * B + row[hh]) * TW + px[hh], v[hh][c]);
            const int voff = 8 * j;
            // first present level of each channel: the three gathers are all
            // issued before any is consumed; further levels (rare) follow
            auto addr = [&](int c, uint32_t pc) -> const VT* {
                const int li = (__ffs(pc) - 1) / 3;
                const int r = li * NR + c * NB + b;
                const int x = s >> (k + li);
                const uint32_t slot = sbase[r] + (uint32_t)__popcll(mask[r] & ((1ull << x) - 1ull));
                return res + (uint64_t)slot * BSQ + voff;
            };
            uint32_t pcs[3];
            int32_t rv[3][8];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                pcs[c] = e.y & (0x249249u << c);             // bits 3i + c: levels k + i
#pragma unroll
                for (int i = 0; i < 8; ++i) rv[c][i] = 0;
                if (pcs[c]) {
                    add8<VT>(addr(c, pcs[c]), rv[c]);
                    pcs[c] &= pcs[c] - 1u;
                }
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                while (pcs[c]) {
                    add8<VT>(addr(c, pcs[c]), rv[c]);
                    pcs[c] &= pcs[c] - 1u;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    v[0][c][i] += rv[c][i];
                    v[1][c][i] += rv[c][4 + i];
                }
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
                ycocg4_pack(v[hh], reinterpret_cast<uint32_t*>(stage + stage_off<B>(S, s, row[hh], px[hh])));
        }
    }
    RLFC_BSTAMP(5);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    RLFC_BSTAMP(6);

    // ---- store ------------------------------------------------------------------------
    const int nrows_band = min(by * B + B, f.height) - by * B;   // rows of this block row
    if (P.store_mode == 2) {
        if (tid == 0) {
            // the output streams through L2 once: for B > 4 evict it first
            // so the record tables, residuals and root colours the other
            // tiles gather stay resident; B = 4 tiles measured faster with
            // the normal policy (P.store_keep)
            uint64_t pol = 0;
            if (P.store_keep)
                asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
            else
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (int st = 0; st < P.nstrip; ++st) {
                const int x0 = (bx0 * B + st * STRIP) * 3;
                if (x0 >= f.width * 3) break;
                asm volatile(
                    "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4}], "
                    "[%5], %6;" ::"l"(&out_map),
                    "r"(x0), "r"((by - P.by_lo) * B), "r"(t), "r"(0), "r"(smem_u32(stage + st * S * B * STRIP * 3)),
                    "l"(pol)
                    : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            RLFC_BSTAMP(7);
        }
    } else {
        // per (view, row, strip): bulk copy when the strip is whole, else bytes
        bool issued = false;
        for (int it = tid; it < S * B * P.nstrip; it += BT) {
            const int st = it % P.nstrip, rr = (it / P.nstrip) % B, s = it / (P.nstrip * B);
            if (rr >= nrows_band) continue;
            const int img = s * T + t;
            const int slot = P.slots ? P.slots[img] : img;
            if (slot < 0) continue;
            const int x0 = bx0 * B + st * STRIP;
            if (x0 >= f.width) continue;
            const int npx = min(STRIP, f.width - x0);
            uint8_t* orow = P.rgb + (int64_t)slot * P.img_stride + (int64_t)((by - P.by_lo) * B + rr) * P.row_stride +
                            (int64_t)x0 * 3;
            const uint8_t* src = stage + stage_off<B>(S, s, rr, st * STRIP);
            if (P.store_mode == 1 && npx == STRIP) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(orow),
                             "r"(smem_u32(src)), "n"(STRIP * 3)
                             : "memory");
                issued = true;
            } else {
                for (int j = 0; j < npx * 3; ++j) orow[j] = src[j];
            }
        }
        if (issued) {
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
    }
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

static bool encode_map(CUtensorMap* map, CUtensorMapDataType dt, cuuint32_t rank, void* base, const cuuint64_t* dims,
                       const cuuint64_t* strides, const cuuint32_t* box) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const cuuint32_t estr[5] = {1u, 1u, 1u, 1u, 1u};
    return enc(map, dt, rank, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Plan {
    BlendParams P;
    int smem;
};

// Blend geometry and shared-memory layout; false when outside the envelope.
template <typename RT>
static bool plan_blend(const rlfc_field& f, int k, bool manual_roots, int tw_first, Plan& pl, bool no_list = false) {
    const int B = f.block, S = f.s_count, h = f.tree_height;
    BlendParams& P = pl.P;
    auto al = [](int x) { return (x + 127) & ~127; };
    const int tws[2] = {tw_first, tw_first == 128 ? 64 : 128};
    for (int TW : tws) {
        if (TW % B) continue;
        const int NB = TW / B;
        if (NB > 64) continue;
        const int NR = 3 * NB, nlev = h - k;
        int off = 0;
        P.off_mbar = off;  off = al(off + 16);
        P.off_flag = off;  off = al(off + NR * 4);
        P.off_mask = off;  off = al(off + nlev * NR * 8);
        P.off_sbase = off; off = al(off + nlev * NR * 4);
        P.off_roots = off; off = al(off + f.rsx * 3 * B * TW * (int)sizeof(RT));
        P.off_rgb = off;   off = al(off + (manual_roots ? f.rsx * B * TW * 3 : 0));
        P.off_cnt = off;   off = al(off + 16);
        P.off_list = off;  off = al(off + (no_list ? 0 : S * NB * 8));
        P.off_stage = off; off = al(off + S * B * TW * 3);
        if (off <= 100 * 1024) {
            P.TW = TW;
            P.NB = NB;
            P.nstrip = TW / STRIP;
            P.nchunks = (f.wb + NB - 1) / NB;
            pl.smem = off;
            return true;
        }
    }
    return false;
}

template <int BSQ, typename VT>
static void run_payloads(const rlfc_field& f, const Ws& w, int by_lo, int by_hi, int sms, cudaStream_t stream,
                         const uint32_t* sel = nullptr) {
    const uint64_t want = (w.cap + PAY_CHUNK - 1) / PAY_CHUNK + 3;
    const uint64_t cap_grid = (uint64_t)sms * 8;
    const unsigned grid = (unsigned)(want < 1 ? 1 : want < cap_grid ? want : cap_grid);
    const int pdyn = BSQ == 16 ? 2 * PAY_BUF : 16;
    cudaFuncSetAttribute(k_payloads<BSQ, VT>, cudaFuncAttributeMaxDynamicSharedMemorySize, pdyn);
    // residual payloads are stored with an L2 evict-last policy so the
    // blend's gathers hit L2
    k_payloads<BSQ, VT><<<grid, THREADS, pdyn, stream>>>(f, w, 1, by_lo, by_hi, sel);
}

template <int B, typename VT, typename RT>
static int launch(const rlfc_field& f, int k, const int32_t* slots, int by_lo, int by_hi, uint8_t* rgb,
                  int64_t img_stride, int64_t row_stride, const Ws& w, int n_flagged, uint64_t* status,
                  cudaStream_t stream, bool build_units = false, const int32_t* trows = nullptr, int ntrows = 0,
                  const uint32_t* sel_dev = nullptr, int sel_n = -1) {
    constexpr int BSQ = B * B;
    const bool tma_ok = w.root_rgb && (reinterpret_cast<uintptr_t>(f.roots) & 15) == 0 &&
                        ((f.wp * (int)sizeof(RT)) % 16) == 0 && encode_fn() != nullptr;
    // blend CTA shape: 96 threads on 64-pixel tiles. Tile residency is what
    // bounds the blend (output bytes in flight / tile lifetime): at 64
    // registers, 96-thread CTAs fit 10 per SM (shared memory 10 x 22.6 KB)
    // against 8 for 128 threads (455 vs 448 Gpix/s)
#ifndef RLFC_DENSE_FRAC
#define RLFC_DENSE_FRAC 0.12      // present nodes / (records x nodes): R4 0.064, R5 0.21, R6 0.40
#endif
#ifndef RLFC_BLEND_BT
#define RLFC_BLEND_BT 96
#define RLFC_BLEND_TW 64
#endif
    constexpr int bt = RLFC_BLEND_BT, tw = RLFC_BLEND_TW;     // compile-time (tools/variant_sweep.py)
    Plan pl{};
    // with the prepared dirty-unit lists (B = 4, 64-pixel tiles) the shared
    // pair list is not needed: a smaller tile fits more CTAs per SM
    const bool lists = B == 4 && w.units && !build_units;
    if (!plan_blend<RT>(f, k, !tma_ok, tw, pl, lists)) return RLFC_ERR_ARGUMENT;
    if (lists && pl.P.NB != 16 && !plan_blend<RT>(f, k, !tma_ok, tw, pl, false)) return RLFC_ERR_ARGUMENT;
    BlendParams& P = pl.P;
    P.f = f;
    P.k = k;
    P.slots = slots;
    P.by_lo = by_lo;
    P.rgb = rgb;
    P.img_stride = img_stride;
    P.row_stride = row_stride;
    P.status = status;
    P.rec_base = w.rec_base;
    P.rec_flag = w.rec_flag;
    P.res = w.res;
    P.root_rgb_g = w.root_rgb;
    P.rgb_stride = w.rgb_stride;
    P.bm = w.bm;
    P.rk = w.rk;
    P.nwp = w.nwp;
    P.roots_vec = ((f.wp * (int)sizeof(RT)) % 16) == 0 && (reinterpret_cast<uintptr_t>(f.roots) & 15) == 0;
    P.trows = trows && !build_units ? trows : nullptr;
    P.units = B == 4 && P.NB == 16 ? w.units : nullptr;
    P.ucap = w.ucap;
    P.build_units = build_units && P.units ? 1 : 0;
    if (build_units && !P.units) return RLFC_OK;
    const int h = f.tree_height, S = f.s_count;
    // output path
    const bool aligned = ((reinterpret_cast<uintptr_t>(rgb) | (uintptr_t)img_stride | (uintptr_t)row_stride) & 15) == 0;
    CUtensorMap out_map, rgb_map, root_map;
    memset(&out_map, 0, sizeof(out_map));
    memset(&rgb_map, 0, sizeof(rgb_map));
    memset(&root_map, 0, sizeof(root_map));
    P.store_mode = aligned ? 1 : 0;
    // output L2 policy (TMA stores), measured at cfg2: B = 4 tiles are
    // faster with the normal policy (R4 0.419 vs 0.431 ms, R3 and R6 equal),
    // B = 8 and 16 with evict-first (R2 0.294 vs 0.307 ms, R1 0.168 vs
    // 0.176 ms)
#ifndef RLFC_STORE_KEEP_B
#define RLFC_STORE_KEEP_B 4
#endif
    P.store_keep = B <= RLFC_STORE_KEEP_B ? 1 : 0;
    const int nrows = min(by_hi * B, f.height) - by_lo * B;
    if (aligned && !slots && S <= 256) {
        const cuuint64_t dims[4] = {(cuuint64_t)f.width * 3, (cuuint64_t)nrows, (cuuint64_t)f.t_count,
                                    (cuuint64_t)S};
        const cuuint64_t strides[3] = {(cuuint64_t)row_stride, (cuuint64_t)img_stride,
                                       (cuuint64_t)img_stride * f.t_count};
        const cuuint32_t box[4] = {(cuuint32_t)(STRIP * 3), (cuuint32_t)B, 1u, (cuuint32_t)S};
        if (encode_map(&out_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, rgb, dims, strides, box)) P.store_mode = 2;
    }
    // input path: RGB(root) rows + raw roots by TMA when the layouts allow it
    P.tma_in = 0;
    const int nroot = f.rsx * f.rsy;
    if (tma_ok) {
        const cuuint64_t d1[3] = {(cuuint64_t)f.wp * 3, (cuuint64_t)f.hp, (cuuint64_t)nroot};
        const cuuint64_t s1[2] = {(cuuint64_t)w.rgb_stride, (cuuint64_t)w.rgb_stride * f.hp};
        const cuuint32_t b1[3] = {(cuuint32_t)(STRIP * 3), (cuuint32_t)B, 1u};
        const cuuint64_t d2[3] = {(cuuint64_t)f.wp, (cuuint64_t)f.hp, (cuuint64_t)nroot * 3};
        const cuuint64_t s2[2] = {(cuuint64_t)f.wp * sizeof(RT), (cuuint64_t)f.wp * f.hp * sizeof(RT)};
        const cuuint32_t b2[3] = {(cuuint32_t)P.TW, (cuuint32_t)B, 1u};
        if (encode_map(&rgb_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, w.root_rgb, d1, s1, b1) &&
            encode_map(&root_map, sizeof(RT) == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_INT32,
                       3, const_cast<void*>(f.roots), d2, s2, b2))
            P.tma_in = 1;
        else
            return RLFC_ERR_ARGUMENT;        // planned without the manual root buffers
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // Programmatic dependent launch: k_blend's CTAs start their TMA loads and
    // record-table loads while k_payloads drains.
    constexpr bool pdl = true;
    cudaLaunchAttribute pdl_attr[1];
    pdl_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl_attr[0].val.programmaticStreamSerializationAllowed = 1;
    auto cfg_of = [&](dim3 g, dim3 b, size_t smem, bool programmatic) {
        cudaLaunchConfig_t c{};
        c.gridDim = g;
        c.blockDim = b;
        c.dynamicSmemBytes = smem;
        c.stream = stream;
        c.attrs = programmatic && pdl ? pdl_attr : nullptr;
        c.numAttrs = programmatic && pdl ? 1 : 0;
        return c;
    };
    if (P.build_units) P.tma_in = 0;
    if (k < h && !P.build_units) {
        // a slot-mode decode of few views decodes only their chain nodes;
        // the full pass then exits at once (and runs when there are more)
        // (a caller that built the node list on the host passes it in
        // device memory with its count: no k_sel_nodes, and no launch of the
        // full pass when the list is in use)
        const bool sel = slots != nullptr && (w.sel != nullptr || sel_dev != nullptr);
        const uint32_t* selp = sel_dev ? sel_dev : w.sel;
        const bool host_sel = sel && sel_dev != nullptr;
        bool full = true;
        if (sel) {
            if (!host_sel) k_sel_nodes<<<1, 256, 0, stream>>>(f, slots, k, w.sel);
            const int64_t nrb = 3ll * (by_hi - by_lo) * f.wb;
            const bool use = !host_sel || (sel_n > 0 && sel_n <= SEL_MAX);
            if (nrb > 0 && use)
                k_payloads_sel<BSQ, VT><<<(unsigned)((nrb + THREADS - 1) / THREADS), THREADS, 0, stream>>>(
                    f, w, by_lo, by_hi, selp);
            if (host_sel) full = !use;
        }
        if (full) run_payloads<BSQ, VT>(f, w, by_lo, by_hi, sms, stream, sel && !host_sel ? w.sel : nullptr);
    }
    // dense streams (many units with several present levels): the variant
    // holding three levels per unit in registers
    const double density = (double)w.cap / ((double)3 * f.wb * f.hb * f.m_nodes);
    auto kern = B == 4 && sizeof(VT) == 2 && density > RLFC_DENSE_FRAC ? k_blend<B, VT, RT, bt, RLFC_DENSE_NL>
                                                                        : k_blend<B, VT, RT, bt, 1>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
    // tile residency is bounded by shared memory: ask for the largest carveout
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const dim3 grid((unsigned)P.nchunks, (unsigned)(P.trows ? ntrows : f.t_count), (unsigned)(by_hi - by_lo));
    if (grid.y == 0) return RLFC_OK;
    {
        const cudaLaunchConfig_t c = cfg_of(grid, dim3(bt), pl.smem, k < h && !P.build_units);
        cudaLaunchKernelEx(&c, kern, P, out_map, rgb_map, root_map);
    }
    if (n_flagged > 0 && k < h && !P.build_units) {
        const int nv = f.s_count * f.t_count;
        k_fixup<B><<<dim3((unsigned)n_flagged, (unsigned)((nv + 63) / 64)), 64, 0, stream>>>(
            f, w.flist, k, slots, by_lo, by_hi, rgb, img_stride, row_stride, status);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "rlfc_b200: staged decode launch error: %s\n", cudaGetErrorString(e));
        return RLFC_ERR_CUDA;
    }
    return RLFC_OK;
}

static bool in_envelope(const rlfc_field& f) {
    if (f.tree_height < 1 || f.tree_height > MAXH || f.s_count > MAXS || f.t_count > 65535) return false;
    if (f.quant_shift < 0 || f.quant_shift > 20) return false;    // dequantised codes fit int32
    if (f.block != 4 && f.block != 8 && f.block != 16) return false;
    for (int l = 0; l < f.tree_height; ++l)
        if (f.level_sx[l] > 64) return false;
    if ((int64_t)f.wb * f.hb >= (1ll << 25)) return false;        // entry block field
    for (int c = 0; c < 3; ++c)
        if (f.srv_len[c] >= (1ull << 32) - 64) return false;      // 32-bit payload offsets
    return true;
}

}  // namespace staged
}  // namespace rlfc

using namespace rlfc;

#ifdef RLFC_BLEND_TIMING
extern "C" int rlfc_debug_blend(long long* host_out) {
    return cudaMemcpyFromSymbol(host_out, staged::g_btime, sizeof(staged::g_btime)) == cudaSuccess ? 0 : 4;
}
#endif

extern "C" int rlfc_count_present(const rlfc_field* f, uint64_t* count, void* stream) {
    if (!f || !count) return RLFC_ERR_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaMemsetAsync(count, 0, 8, s);
    const int64_t nrec = 3ll * f->wb * f->hb;
    if (nrec > 0)
        staged::k_count_present<<<(unsigned)((nrec + 255) / 256), 256, 0, s>>>(
            *f, reinterpret_cast<unsigned long long*>(count));
    return cudaGetLastError() == cudaSuccess ? RLFC_OK : RLFC_ERR_CUDA;
}

extern "C" int rlfc_decode_workspace_bytes(const rlfc_field* f, uint64_t present_total, uint64_t* bytes) {
    if (!f || !bytes) return RLFC_ERR_ARGUMENT;
    *bytes = staged::carve(*f, nullptr, present_total, nullptr);
    return staged::in_envelope(*f) ? RLFC_OK : RLFC_ERR_ARGUMENT;
}

extern "C" int rlfc_staged_prepare(const rlfc_field* f, void* workspace, uint64_t workspace_bytes,
                                   uint64_t present_total, int32_t* n_flagged, void* stream) {
    if (!f || !workspace) return RLFC_ERR_ARGUMENT;
    if (!staged::in_envelope(*f)) return RLFC_ERR_ARGUMENT;
    staged::Ws w;
    if (staged::carve(*f, workspace, present_total, &w) > workspace_bytes) return RLFC_ERR_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0) return RLFC_ERR_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t nrec = 3ll * f->wb * f->hb;
    cudaMemsetAsync(w.counter, 0, 8, s);
    if (nrec > 0) {
        staged::k_rec_count<<<(unsigned)((nrec + 255) / 256), 256, 0, s>>>(*f, w.rec_base);
        {
            // the anomaly list (written last) holds the partial sums meanwhile
            const int64_t nparts = (nrec + staged::SCAN_TILE - 1) / staged::SCAN_TILE;
            staged::k_scan_part<<<(unsigned)nparts, 256, 0, s>>>(w.rec_base, nrec, w.flist);
            staged::k_scan_bases<<<1, 1024, 0, s>>>(w.flist, nparts, w.counter);
            staged::k_scan_apply<<<(unsigned)nparts, 256, 0, s>>>(w.rec_base, nrec, w.flist);
        }
        const unsigned g = (unsigned)((nrec + staged::THREADS - 1) / staged::THREADS);
        switch (f->block) {
            case 4: staged::k_index<16><<<g, staged::THREADS, 0, s>>>(*f, 0, 0, f->hb, w, w.rec_base); break;
            case 8: staged::k_index<64><<<g, staged::THREADS, 0, s>>>(*f, 0, 0, f->hb, w, w.rec_base); break;
            default: staged::k_index<256><<<g, staged::THREADS, 0, s>>>(*f, 0, 0, f->hb, w, w.rec_base); break;
        }
    }
    if (present_total > 0)
        staged::k_sort_chunks<<<(unsigned)((present_total + staged::PAY_CHUNK - 1) / staged::PAY_CHUNK),
                                staged::THREADS, 0, s>>>(w, present_total);
    // every payload decoded once here too: corrupt packs flag their records
    // (kernels.py:147-150), so the anomaly list below is complete
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const bool small = f->quant_shift <= 4;
        switch (f->block) {
            case 4: small ? staged::run_payloads<16, int16_t>(*f, w, 0, f->hb, sms, s)
                          : staged::run_payloads<16, int32_t>(*f, w, 0, f->hb, sms, s); break;
            case 8: small ? staged::run_payloads<64, int16_t>(*f, w, 0, f->hb, sms, s)
                          : staged::run_payloads<64, int32_t>(*f, w, 0, f->hb, sms, s); break;
            default: small ? staged::run_payloads<256, int16_t>(*f, w, 0, f->hb, sms, s)
                           : staged::run_payloads<256, int32_t>(*f, w, 0, f->hb, sms, s); break;
        }
    }
    cudaMemsetAsync(w.flist, 0, 4, s);
    if (nrec > 0) staged::k_flag_list<<<(unsigned)((nrec + 255) / 256), 256, 0, s>>>(w.rec_flag, nrec, w.flist);
    uint32_t nf = 0;
    cudaMemcpyAsync(&nf, w.flist, 4, cudaMemcpyDeviceToHost, s);
    // the B = 4 blend's dirty-unit lists (stream-invariant: presence bits and
    // anomaly flags only), built by the blend's own record phase and pair scan
    if (f->block == 4 && w.units) {
        const int rc = f->roots_i16 ? (f->quant_shift <= 4 ? staged::launch<4, int16_t, int16_t>(
                                           *f, 0, nullptr, 0, f->hb, nullptr, 0, 0, w, 0, nullptr, s, true)
                                                           : staged::launch<4, int32_t, int16_t>(
                                           *f, 0, nullptr, 0, f->hb, nullptr, 0, 0, w, 0, nullptr, s, true))
                                    : (f->quant_shift <= 4 ? staged::launch<4, int16_t, int32_t>(
                                           *f, 0, nullptr, 0, f->hb, nullptr, 0, 0, w, 0, nullptr, s, true)
                                                           : staged::launch<4, int32_t, int32_t>(
                                           *f, 0, nullptr, 0, f->hb, nullptr, 0, 0, w, 0, nullptr, s, true));
        if (rc != RLFC_OK) return rc;
    }
    const bool tma_ok = (reinterpret_cast<uintptr_t>(f->roots) & 15) == 0 &&
                        ((f->wp * (f->roots_i16 ? 2 : 4)) % 16) == 0;
    if (tma_ok) {
        const int64_t n = (int64_t)f->rsx * f->rsy * f->hp * (f->wp / 4);
        const int64_t want = (n + staged::THREADS - 1) / staged::THREADS;
        const unsigned g = (unsigned)(want < 148 * 16 ? want : 148 * 16);
        if (f->roots_i16)
            staged::k_root_rgb<int16_t><<<g, staged::THREADS, 0, s>>>(*f, w.root_rgb, w.rgb_stride, 0, f->hp);
        else
            staged::k_root_rgb<int32_t><<<g, staged::THREADS, 0, s>>>(*f, w.root_rgb, w.rgb_stride, 0, f->hp);
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) return RLFC_ERR_CUDA;
    if (n_flagged) *n_flagged = (int32_t)nf;
    return cudaGetLastError() == cudaSuccess ? RLFC_OK : RLFC_ERR_CUDA;
}

extern "C" int rlfc_staged_index_view(const rlfc_field* f, void* workspace, uint64_t workspace_bytes,
                                      uint64_t present_total, rlfc_index_view* out) {
    if (!f || !workspace || !out) return RLFC_ERR_ARGUMENT;
    if (!staged::in_envelope(*f)) return RLFC_ERR_ARGUMENT;
    staged::Ws w;
    if (staged::carve(*f, workspace, present_total, &w) > workspace_bytes) return RLFC_ERR_ARGUMENT;
    out->bm = w.bm;
    out->rk = w.rk;
    out->rec_flag = w.rec_flag;
    out->entries = reinterpret_cast<const uint32_t*>(w.entries);
    out->nrec = 3ll * f->wb * f->hb;
    out->nwp = w.nwp;
    out->_pad = 0;
    out->cap = w.cap;
    return RLFC_OK;
}

extern "C" int rlfc_decode_blocks_indexed(const rlfc_field* f, void* workspace, uint64_t workspace_bytes,
                                          uint64_t present_total, const int32_t* req, int32_t n, int32_t* out,
                                          int32_t* status, void* stream) {
    if (!f || !workspace || n < 0) return RLFC_ERR_ARGUMENT;
    if (!staged::in_envelope(*f)) return RLFC_ERR_ARGUMENT;
    staged::Ws w;
    if (staged::carve(*f, workspace, present_total, &w) > workspace_bytes) return RLFC_ERR_ARGUMENT;
    if (n == 0) return RLFC_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned g = (unsigned)((n + 127) / 128);
    switch (f->block) {
        case 4: staged::k_blocks_indexed<4><<<g, 128, 0, s>>>(*f, w, req, n, out, status); break;
        case 8: staged::k_blocks_indexed<8><<<g, 128, 0, s>>>(*f, w, req, n, out, status); break;
        case 16: staged::k_blocks_indexed<16><<<g, 128, 0, s>>>(*f, w, req, n, out, status); break;
        default: return RLFC_ERR_ARGUMENT;
    }
    return cudaGetLastError() == cudaSuccess ? RLFC_OK : RLFC_ERR_CUDA;
}

extern "C" int rlfc_decode_field_staged(const rlfc_field* f, int32_t stop_level, const int32_t* image_slots,
                                        int32_t by_lo, int32_t by_hi, uint8_t* rgb, int64_t img_stride,
                                        int64_t row_stride, void* workspace, uint64_t workspace_bytes,
                                        uint64_t present_total, int32_t n_flagged, const int32_t* t_rows,
                                        int32_t n_trows, uint64_t* status, void* stream) {
    return rlfc::decode_field_staged_sel(f, stop_level, image_slots, by_lo, by_hi, rgb, img_stride, row_stride,
                                         workspace, workspace_bytes, present_total, n_flagged, t_rows, n_trows,
                                         status, stream, nullptr, -1);
}

namespace rlfc {
int sel_nodes_host(const rlfc_field& f, int k, const int32_t* views, int nviews, uint32_t* out) {
    // the distinct chain nodes at levels >= k of the given views (serial
    // indices), ascending (k_sel_nodes on the host): out[0] = count, or
    // SEL_MAX + 1 when there are more
    uint32_t nodes[staged::SEL_MAX];
    int n = 0;
    for (int i = 0; i < nviews; ++i) {
        const int s = views[i] / f.t_count, t = views[i] % f.t_count;
        for (int l = k; l < f.tree_height; ++l) {
            const uint32_t nd = (uint32_t)(f.level_base[l] + (t >> l) * f.level_sx[l] + (s >> l));
            bool seen = false;
            for (int j = 0; j < n && !seen; ++j) seen = nodes[j] == nd;
            if (seen) continue;
            if (n == staged::SEL_MAX) {
                out[0] = staged::SEL_MAX + 1;
                return staged::SEL_MAX + 1;
            }
            nodes[n++] = nd;
        }
    }
    std::sort(nodes, nodes + n);
    out[0] = (uint32_t)n;
    for (int j = 0; j < n; ++j) out[1 + j] = nodes[j];
    return n;
}

int decode_field_staged_sel(const rlfc_field* f, int32_t stop_level, const int32_t* image_slots, int32_t by_lo,
                            int32_t by_hi, uint8_t* rgb, int64_t img_stride, int64_t row_stride, void* workspace,
                            uint64_t workspace_bytes, uint64_t present_total, int32_t n_flagged,
                            const int32_t* t_rows, int32_t n_trows, uint64_t* status, void* stream,
                            const uint32_t* sel_dev, int sel_n) {
    if (!f || !rgb || !status || !workspace) return RLFC_ERR_ARGUMENT;
    if (stop_level < 0 || stop_level > f->tree_height || by_lo < 0 || by_hi > f->hb || by_lo > by_hi)
        return RLFC_ERR_ARGUMENT;
    if (!staged::in_envelope(*f)) return RLFC_ERR_ARGUMENT;
    if (by_lo == by_hi) return RLFC_OK;
    staged::Ws w;
    if (staged::carve(*f, workspace, present_total, &w) > workspace_bytes) return RLFC_ERR_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0) return RLFC_ERR_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool small = f->quant_shift <= 4, r16 = f->roots_i16 != 0;
#define RLFC_STAGED(B_)                                                                                            \
    if (small && r16)                                                                                              \
        return staged::launch<B_, int16_t, int16_t>(*f, stop_level, image_slots, by_lo, by_hi, rgb, img_stride,   \
                                                    row_stride, w, n_flagged, status, s, false, t_rows, n_trows,  \
                                                    sel_dev, sel_n);                                     \
    if (small)                                                                                                     \
        return staged::launch<B_, int16_t, int32_t>(*f, stop_level, image_slots, by_lo, by_hi, rgb, img_stride,   \
                                                    row_stride, w, n_flagged, status, s, false, t_rows, n_trows,  \
                                                    sel_dev, sel_n);                                     \
    if (r16)                                                                                                       \
        return staged::launch<B_, int32_t, int16_t>(*f, stop_level, image_slots, by_lo, by_hi, rgb, img_stride,   \
                                                    row_stride, w, n_flagged, status, s, false, t_rows, n_trows,  \
                                                    sel_dev, sel_n);                                     \
    return staged::launch<B_, int32_t, int32_t>(*f, stop_level, image_slots, by_lo, by_hi, rgb, img_stride,       \
                                                row_stride, w, n_flagged, status, s, false, t_rows, n_trows,  \
                                                    sel_dev, sel_n);
    switch (f->block) {
        case 4: { RLFC_STAGED(4) }
        case 8: { RLFC_STAGED(8) }
        case 16: { RLFC_STAGED(16) }
        default: return RLFC_ERR_ARGUMENT;
    }
#undef RLFC_STAGED
}
}  // namespace rlfc
