// rlfc_common.cuh -- device helpers shared by the RLFC decode / render kernels.
//
// Everything here is integer-only and bit-exact with the reference kernels
// (/root/reference/pkg/src/rlfc/kernels.py).  Payload bits are LSB-first
// across bytes (kernels.py:1-11); every value of a BISE payload has a
// closed-form bit offset because all groups but the last are full
// (SURVEY.md Appendix A), so no per-value prefix sum is needed.
#pragma once

#include <cstdint>
#include "../../include/rlfc_b200.h"

namespace rlfc {

constexpr int MODE_BITS = 0;   // kernels.py:17-19
constexpr int MODE_TRIT = 1;
constexpr int MODE_QUINT = 2;
constexpr int NUM_DESC = 30;   // bise.py:22-25

// bise.py:22-60 RANGE_TABLE factored into (mode, low bits) per descriptor
// (TABLE_MODE / TABLE_BITS, bise.py:59-60), packed into 64-bit immediates so
// a lookup is a shift + mask in registers (no memory table).
constexpr uint64_t MODE_PACK = []() constexpr {
    uint64_t v = 0;
    const int m[30] = {0, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0,
                       2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0};
    for (int d = 0; d < 30; ++d) v |= (uint64_t)m[d] << (2 * d);
    return v;
}();
constexpr uint64_t BITS_LO = []() constexpr {   // descriptors 0..15
    const int b[16] = {1, 0, 2, 0, 1, 3, 1, 2, 4, 2, 3, 5, 3, 4, 6, 4};
    uint64_t v = 0;
    for (int d = 0; d < 16; ++d) v |= (uint64_t)b[d] << (4 * d);
    return v;
}();
constexpr uint64_t BITS_HI = []() constexpr {   // descriptors 16..29
    const int b[14] = {5, 7, 5, 6, 8, 6, 7, 9, 7, 8, 10, 8, 9, 11};
    uint64_t v = 0;
    for (int d = 0; d < 14; ++d) v |= (uint64_t)b[d] << (4 * d);
    return v;
}();
__host__ __device__ constexpr int desc_mode(int d) { return (int)((MODE_PACK >> (2 * d)) & 3u); }
__host__ __device__ constexpr int desc_bits(int d) {
    return d < 16 ? (int)((BITS_LO >> (4 * d)) & 15u) : (int)((BITS_HI >> (4 * (d - 16))) & 15u);
}
static_assert(desc_mode(3) == 2 && desc_bits(29) == 11 && desc_bits(17) == 7 && desc_bits(15) == 4, "table");

// kernels.py:63-70 payload_bits
__host__ __device__ constexpr int payload_bits(int mode, int bits, int count) {
    return mode == MODE_BITS ? count * bits
         : mode == MODE_TRIT ? 8 * ((count + 4) / 5) + count * bits
                             : 7 * ((count + 2) / 3) + count * bits;
}
__host__ __device__ constexpr int payload_bytes(int d, int count) {
    return (payload_bits(desc_mode(d), desc_bits(d), count) + 7) >> 3;
}

// Bytes occupied by one present node (descriptor + padded payload) for
// descriptor d at B*B values; index 30 = invalid descriptor sentinel.
struct NodeBytes {
    uint16_t v[32];
};
template <int BSQ>
__host__ __device__ constexpr NodeBytes make_node_bytes() {
    NodeBytes nb{};
    for (int d = 0; d < NUM_DESC; ++d) nb.v[d] = (uint16_t)(1 + payload_bytes(d, BSQ));
    nb.v[30] = 0;
    nb.v[31] = 0;
    return nb;
}

// Packed base-3 / base-5 digit tables (kernels.py:47-60 TRIT_DIGITS /
// QUINT_DIGITS): trit digit i of pack p = (TRIT[p] >> 2i) & 3, quint digit i
// = (QUINT[p] >> 3i) & 7.
struct DigitLut {
    uint16_t trit[243];
    uint16_t quint[125];
};
__host__ __device__ constexpr DigitLut make_digit_lut() {
    DigitLut L{};
    for (int p = 0; p < 243; ++p) {
        int r = p, v = 0;
        for (int i = 0; i < 5; ++i) { v |= (r % 3) << (2 * i); r /= 3; }
        L.trit[p] = (uint16_t)v;
    }
    for (int p = 0; p < 125; ++p) {
        int r = p, v = 0;
        for (int i = 0; i < 3; ++i) { v |= (r % 5) << (3 * i); r /= 5; }
        L.quint[p] = (uint16_t)v;
    }
    return L;
}

// 32 bits starting at absolute bit position `bitpos` of byte array `base`.
// Reads the two aligned 32-bit words covering the position; the buffer must
// be readable 8 bytes past the last payload byte (device SRV copies carry
// >= 16 bytes of zero padding).
// GEN: generic loads (the bytes may sit in shared memory), else read-only
// global loads.
template <bool GEN = false>
__device__ __forceinline__ uint32_t load_bits32(const uint8_t* base, uint64_t bitpos) {
    uintptr_t a = reinterpret_cast<uintptr_t>(base) + (bitpos >> 3);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    uint32_t sh = (uint32_t)((a & 3) << 3) + (uint32_t)(bitpos & 7);
    uint32_t lo, hi;
    if (GEN) {
        lo = w[0];
        hi = w[1];
    } else {
        lo = __ldg(w);
        hi = __ldg(w + 1);
    }
    return __funnelshift_r(lo, hi, sh);
}
template <bool GEN = false>
__device__ __forceinline__ uint32_t get_bits(const uint8_t* base, uint64_t bitpos, int nbits) {
    return load_bits32<GEN>(base, bitpos) & ((1u << nbits) - 1u);
}

// Dequantise one zigzag code (bise.py:69-72 unzigzag + hierarchy.py:232-237
// dequantize, inlined exactly as kernels.py:202-211).  The reference adds in
// int64 and stores into an int32 accumulator; the 32-bit wrap below is the
// same result.
__device__ __forceinline__ int32_t dequant(uint32_t z, int shift) {
    if (z == 0) return 0;
    int64_t half = (int64_t(1) << shift) >> 1;
    int64_t mag = (int64_t)((z + 1) >> 1) << shift;
    int64_t v = (z & 1) ? -(mag + half) : (mag + half);
    return (int32_t)(uint32_t)(uint64_t)v;
}

// kernels.py:128-159 bise_decode_core for one payload, accumulating the
// dequantised values into acc[0..BSQ).  Returns 0 or 1 (corrupt pack).  The
// whole payload is validated before any value is added, as the reference
// decodes into tmp first.
template <int BSQ, bool GEN = false>
__device__ int decode_payload_acc(const uint8_t* p, int desc, int shift, int32_t* acc,
                                  const DigitLut& lut) {
    const int mode = desc_mode(desc), b = desc_bits(desc);
    if (mode != MODE_BITS) {
        const int G = mode == MODE_TRIT ? 5 : 3;
        const int PB = mode == MODE_TRIT ? 8 : 7;
        const uint32_t PMAX = mode == MODE_TRIT ? 242u : 124u;
        const int gbits = PB + G * b;
        for (int g = 0; g * G < BSQ; ++g)
            if (get_bits<GEN>(p, (uint64_t)g * gbits, PB) > PMAX) return 1;
    }
    for (int k = 0; k < BSQ; ++k) {
        uint32_t z;
        if (mode == MODE_BITS) {
            z = get_bits<GEN>(p, (uint64_t)k * b, b);
        } else if (mode == MODE_TRIT) {
            int g = k / 5, i = k - 5 * g;
            uint64_t gp = (uint64_t)g * (8 + 5 * b);
            uint32_t pack = get_bits<GEN>(p, gp, 8);
            uint32_t digit = (lut.trit[pack] >> (2 * i)) & 3u;
            uint32_t low = b ? get_bits<GEN>(p, gp + 8 + i * b, b) : 0u;
            z = (digit << b) | low;
        } else {
            int g = k / 3, i = k - 3 * g;
            uint64_t gp = (uint64_t)g * (7 + 3 * b);
            uint32_t pack = get_bits<GEN>(p, gp, 7);
            uint32_t digit = (lut.quint[pack] >> (3 * i)) & 7u;
            uint32_t low = b ? get_bits<GEN>(p, gp + 7 + i * b, b) : 0u;
            z = (digit << b) | low;
        }
        acc[k] += dequant(z, shift);
    }
    return 0;
}

// 32 presence bits of nodes [n0, n0+32) of a record's bitmap (bit i of the
// record = byte i>>3 bit i&7, kernels.py:181-183), n0 a multiple of 32.
template <bool GEN = false>
__device__ __forceinline__ uint32_t bitmap_word(const uint8_t* rec, int n0) {
    return load_bits32<GEN>(rec, (uint64_t)n0);
}

// Node size (descriptor + payload bytes) for B*B = 16 values from three
// 64-bit immediates (5 bits per descriptor): no memory access in a walk's
// dependent chain (k_index, walk_chain).
constexpr uint64_t nb16_word(int w) {
    uint64_t v = 0;
    for (int i = 0; i < 12; ++i) {
        const int d = w * 12 + i;
        if (d < NUM_DESC) v |= (uint64_t)(1 + payload_bytes(d, 16)) << (5 * i);
    }
    return v;
}
__device__ __forceinline__ uint32_t node_bytes16(int d) {
    constexpr uint64_t W0 = nb16_word(0), W1 = nb16_word(1), W2 = nb16_word(2);
    const uint64_t w = d < 12 ? W0 : d < 24 ? W1 : W2;
    const int i = d < 12 ? d : d < 24 ? d - 12 : d - 24;
    return (uint32_t)(w >> (5 * i)) & 31u;
}

// ---- closed-form BISE windows (B = 4, 16 values) -------------------------------------
// kernels.py:202-211 dequantisation in 32-bit wrap arithmetic: identical to
// the reference's int64 result truncated into its int32 accumulator.
__device__ __forceinline__ int32_t deq(uint32_t z, int shift) {
    if (shift >= 32) return dequant(z, shift);
    const uint32_t mag = (((z + 1u) >> 1) << shift) + ((1u << shift) >> 1);
    const uint32_t v = (z & 1u) ? 0u - mag : mag;
    return z ? (int32_t)v : 0;
}

// 64 bits of the aligned words sw from bit pos (generic: shared or global).
__device__ __forceinline__ uint64_t win64(const uint32_t* sw, uint32_t pos) {
    const uint32_t wi = pos >> 5, o = pos & 31u;
    const uint32_t a = sw[wi], b = sw[wi + 1], c = sw[wi + 2];
    return (uint64_t)__funnelshift_r(a, b, o) | (uint64_t)__funnelshift_r(b, c, o) << 32;
}

// decode16 for one request (k_blocks_indexed, k_block_server): the windows read straight
// from the SRV words in memory, digits from the global LUT, dequantisation
// by arithmetic, accumulated into acc (kernels.py:128-159, 202-211).
template <int MODE>
__device__ __forceinline__ bool decode16_acc(const uint32_t* sw, uint32_t bit0, uint32_t b, const uint16_t* dlut,
                                             int shift, int32_t* acc) {
    const uint32_t lm = (1u << b) - 1u;
    bool bad = false;
    if (MODE == MODE_BITS) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t w = win64(sw, bit0 + 4u * (uint32_t)q * b);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[4 * q + i] += deq((uint32_t)(w >> ((uint32_t)i * b)) & lm, shift);
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
            const uint32_t dg = __ldg(dlut + (pk <= PMAX ? pk : 0u));
#pragma unroll
            for (int i = 0; i < G && g * G + i < 16; ++i) {
                const uint32_t low = (uint32_t)(w >> (PB + (uint32_t)i * b)) & lm;
                acc[g * G + i] += deq((((dg >> (DB * i)) & DMASK) << b) | low, shift);
            }
        }
    }
    return bad;
}

// Serial index of image (s, t)'s level-l ancestor (container.py:122-145).
__device__ __forceinline__ int chain_node(const rlfc_field& f, int l, int s, int t) {
    return f.level_base[l] + (t >> l) * f.level_sx[l] + (s >> l);
}

// kernels.py:162-216 decode_chain_core: walk one record up to the image's
// last target (levels h-1 .. stop_level), decoding target payloads into acc
// (pre-filled with the root block).  Present nodes are visited with
// find-first-set over the bitmap, so the walk costs one step per PRESENT
// node; the result and the status (0 / 1 / 2) are identical to the
// reference's node-by-node loop.
//
// avail: bytes of the stream readable from rec (the SRV section from the
// record on; bit windows may read 8 bytes further, into the 16-byte
// padding).  A descriptor or payload past avail returns WALK_OOB: the
// reference has no defined behaviour there (numba does not bounds-check),
// and the device must not fault; callers report it as code 2.
constexpr int WALK_OOB = 3;
template <int BSQ, bool GEN = false>
__device__ int walk_chain(const rlfc_field& f, const uint8_t* rec, int s, int t, int stop_level,
                          int32_t* acc, const DigitLut& lut, const NodeBytes& nb, uint64_t avail) {
    const int h = f.tree_height;
    const int nt = h - stop_level;
    if (nt <= 0) return 0;
    if ((uint64_t)f.bitmap_bytes > avail) return WALK_OOB;
    int ti = 0;                                  // next target, level h-1-ti
    int target = chain_node(f, h - 1, s, t);
    const int last = chain_node(f, stop_level, s, t);
    uint64_t cursor = (uint64_t)f.bitmap_bytes;  // relative to rec
    for (int n0 = 0; n0 <= last; n0 += 32) {
        uint32_t bits = bitmap_word<GEN>(rec, n0);
        int span = last - n0 + 1;                // nodes n0..last
        if (span < 32) bits &= (1u << span) - 1u;
        while (bits) {
            int node = n0 + __ffs(bits) - 1;
            bits &= bits - 1u;
            while (target < node) {              // absent targets contribute 0
                if (++ti == nt) return 0;
                target = chain_node(f, h - 1 - ti, s, t);
            }
            if (cursor >= avail) return WALK_OOB;
            int desc = rec[cursor];
            if (desc >= NUM_DESC) return 2;
            const uint32_t nbytes = BSQ == 16 ? node_bytes16(desc) : (uint32_t)nb.v[desc];
            if (cursor + nbytes > avail) return WALK_OOB;
            if (target == node) {
                int st = decode_payload_acc<BSQ, GEN>(rec + cursor + 1, desc, f.quant_shift, acc, lut);
                if (st) return st;
                if (++ti == nt) return 0;
                target = chain_node(f, h - 1 - ti, s, t);
            }
            cursor += nbytes;
        }
    }
    return 0;
}

// Bytes of channel c's SRV section from byte offset off on (0 past the end).
__device__ __forceinline__ uint64_t srv_avail(const rlfc_field& f, int c, uint64_t off) {
    return off < f.srv_len[c] ? f.srv_len[c] - off : 0;
}

__device__ __forceinline__ int32_t root_sample(const rlfc_field& f, int s, int t, int c, int y, int x) {
    const int h = f.tree_height;
    int64_t idx = ((((int64_t)(s >> h) * f.rsy + (t >> h)) * 3 + c) * f.hp + y) * f.wp + x;
    return f.roots_i16 ? (int32_t)reinterpret_cast<const int16_t*>(f.roots)[idx]
                       : reinterpret_cast<const int32_t*>(f.roots)[idx];
}

// colorspace.py:27-36 ycocgr_to_rgb (arithmetic shifts = floor halves)
// followed by colorspace.py:46-56 clip to [0, 255].
__device__ __forceinline__ uint32_t clamp8(int32_t v) { return (uint32_t)min(max(v, 0), 255); }
__device__ __forceinline__ void ycocg_to_rgb8(int32_t y, int32_t co, int32_t cg, uint32_t& r,
                                              uint32_t& g, uint32_t& b) {
    int32_t t = y - (cg >> 1);
    int32_t gg = cg + t;
    int32_t bb = t - (co >> 1);
    int32_t rr = bb + co;
    r = clamp8(rr);
    g = clamp8(gg);
    b = clamp8(bb);
}

// Failure word for the device status (see rlfc_b200.h).
__device__ __forceinline__ void report(uint64_t* status, uint64_t key, int code) {
    if (code) atomicMax((unsigned long long*)status,
                        (unsigned long long)(((RLFC_KEY_MAX - key) << 2) | (uint64_t)code));
}

}  // namespace rlfc
