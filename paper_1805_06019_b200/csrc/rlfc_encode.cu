// rlfc_encode.cu -- RKV/SRV tree construction and record serialisation on
// the GPU (the producer side of the path).
//
// Restates the reference encoder kernel by kernel; every operation is per
// pixel, per block or per record, so each is one thread:
//   k_enc_planes    hierarchy.py:185-193 + colorspace.py:17-24: YCoCg-R of
//                   the input, zero padded to (Hp, Wp);
//   k_enc_pyramid   hierarchy.py:195-212: parent = floor((sum w_i * child_i
//                   + 128) / 256) with the integer cluster weights the host
//                   computes exactly as the reference (producer.py);
//   k_enc_srv       hierarchy.py:216-298, one tree level top-down: residual
//                   against the reconstructed parent, pixel threshold, block
//                   energy and presence, quantise (arithmetic shift of the
//                   magnitude), zigzag (as uint16, bise.py:63-66), range
//                   choice (smallest cardinality above the block maximum,
//                   hierarchy.py:263-265), dequantise and closed-loop
//                   reconstruction written over the level's planes;
//   k_enc_rec_size / k_enc_records  container.py:300-323: per record the
//                   presence bitmap, then descriptor + BISE payload
//                   (kernels.py:92-125 bise_encode_core) of every present
//                   node in BFS order.
// Outputs equal the native C++ producer's and the reference encoder's byte
// for byte (tests/test_gpu_encoder.py).
#include <cuda_runtime.h>
#include <cstdint>

#include "rlfc_common.cuh"

namespace rlfc {
namespace enc {

__constant__ int c_card[NUM_DESC] = {2,   3,   4,   5,   6,   8,   10,  12,  16,   20,   24,   32,   40,   48,  64,
                                     80,  96,  128, 160, 192, 256, 320, 384, 512, 640, 768, 1024, 1280, 1536, 2048};

// rgb: (S*T, H_valid, W, 3); planes: (S*T, 3, hp, wp) int32
__global__ void k_enc_planes(const uint8_t* __restrict__ rgb, int64_t nimg, int W, int hv, int hp, int wp,
                             int32_t* __restrict__ planes) {
    const int64_t plane = (int64_t)hp * wp;
    const int64_t n = nimg * plane;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t img = i / plane, o = i - img * plane;
        const int y = (int)(o / wp), x = (int)(o - (int64_t)y * wp);
        int32_t yy = 0, co = 0, cg = 0;
        if (y < hv && x < W) {
            const uint8_t* px = rgb + ((img * hv + y) * (int64_t)W + x) * 3;
            const int32_t r = px[0], g = px[1], b = px[2];
            co = r - b;
            const int32_t t = b + (co >> 1);
            cg = g - t;
            yy = t + (cg >> 1);
        }
        int32_t* P = planes + img * 3 * plane + o;
        P[0] = yy;
        P[plane] = co;
        P[2 * plane] = cg;
    }
}

// child: (sx, sy, 3, hp, wp); parent: (px, py, 3, hp, wp); w: (px*py, 4)
// member weights in the reference member order (x outer, y inner).
__global__ void k_enc_pyramid(const int32_t* __restrict__ child, int sx, int sy, int32_t* __restrict__ parent, int px,
                              int py, const int64_t* __restrict__ w, int64_t plane) {
    const int64_t n = (int64_t)px * py * 3 * plane;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pc = i / plane, o = i - pc * plane;
        const int c = (int)(pc % 3);
        const int cell = (int)(pc / 3), cx = cell / py, cy = cell - cx * py;
        const int64_t* wc = w + (int64_t)cell * 4;
        int64_t acc = 0;
        int m = 0;
        for (int x = 2 * cx; x <= 2 * cx + 1; ++x)
            for (int y = 2 * cy; y <= 2 * cy + 1; ++y)
                if (x < sx && y < sy) acc += wc[m++] * (int64_t)child[(((int64_t)x * sy + y) * 3 + c) * plane + o];
        parent[i] = (int32_t)((acc + 128) >> 8);
    }
}

// One tree level: planes (sx, sy, 3, hp, wp) in: RKV views, out:
// reconstructed views; above: the level above's reconstruction.  desc:
// [3][nblk][M] (0xFF absent, else range index); zv: [3][nblk][M][B*B].
template <int B>
__global__ void k_enc_srv(int32_t* __restrict__ planes, const int32_t* __restrict__ above, int sx, int sy, int psy,
                          int hp, int wp, int pt, int64_t bt, int shift, int level_base, int M,
                          uint8_t* __restrict__ desc, uint16_t* __restrict__ zv, unsigned long long* present,
                          int* err) {
    constexpr int BSQ = B * B;
    const int wb = wp / B, hb = hp / B;
    const int64_t nblk = (int64_t)wb * hb, plane = (int64_t)hp * wp;
    const int64_t n = (int64_t)sx * sy * 3 * nblk;
    const int32_t half = shift > 0 ? (1 << (shift - 1)) : 0;
    unsigned long long npres = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t blk = i % nblk, job = i / nblk;
        const int c = (int)(job % 3), cell = (int)(job / 3), x = cell / sy, y = cell - x * sy;
        const int by = (int)(blk / wb), bx = (int)(blk - (int64_t)by * wb);
        int32_t* ch = planes + ((int64_t)cell * 3 + c) * plane;
        const int32_t* pa = above + (((int64_t)(x / 2) * psy + y / 2) * 3 + c) * plane;
        int32_t q[BSQ];
        int64_t energy = 0;
        for (int yy = 0; yy < B; ++yy)
            for (int xx = 0; xx < B; ++xx) {
                const int64_t o = (int64_t)(by * B + yy) * wp + bx * B + xx;
                int32_t v = ch[o] - pa[o];
                if (abs(v) < pt) v = 0;
                energy += abs(v);
                const int32_t a = abs(v) >> shift;
                q[yy * B + xx] = v < 0 ? -a : a;
            }
        const bool pres = energy >= bt && energy > 0;
        const int node = level_base + y * sx + x;
        const int64_t rec = (int64_t)c * nblk + blk;
        if (pres) {
            uint16_t* z = zv + (rec * M + node) * BSQ;
            uint32_t zmax = 0;
            for (int k = 0; k < BSQ; ++k) {
                const int64_t zz = q[k] >= 0 ? 2 * (int64_t)q[k] : -2 * (int64_t)q[k] - 1;
                const uint16_t z16 = (uint16_t)(uint32_t)zz;
                z[k] = z16;
                zmax = max(zmax, (uint32_t)z16);
            }
            int d = 0;
            while (d < NUM_DESC && c_card[d] <= (int)zmax) ++d;
            if (d == NUM_DESC) {
                atomicExch(err, 1);                // value outside the range table
                d = NUM_DESC - 1;
            }
            desc[rec * M + node] = (uint8_t)d;
            ++npres;
        }
        for (int yy = 0; yy < B; ++yy)
            for (int xx = 0; xx < B; ++xx) {
                const int64_t o = (int64_t)(by * B + yy) * wp + bx * B + xx;
                const int32_t qq = q[yy * B + xx];
                int32_t rh = 0;
                if (pres && qq != 0) {
                    const int32_t mag = ((qq < 0 ? -qq : qq) << shift) + half;
                    rh = qq < 0 ? -mag : mag;
                }
                ch[o] = pa[o] + rh;
            }
    }
    for (int o = 16; o > 0; o >>= 1) npres += __shfl_xor_sync(0xffffffffu, npres, o);
    if ((threadIdx.x & 31) == 0 && npres) atomicAdd(present, npres);
}

__global__ void k_enc_rec_size(const uint8_t* __restrict__ desc, int64_t nrec, int M, int bsq,
                               uint64_t* __restrict__ size) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrec) return;
    uint64_t sz = (uint64_t)(M + 7) >> 3;
    const uint8_t* d = desc + r * M;
    for (int n = 0; n < M; ++n)
        if (d[n] != 0xFF) sz += 1 + (uint64_t)payload_bytes(d[n], bsq);
    size[r] = sz;
}

// LSB-first bit writer (kernels.py:73-80 put_bits) into pre-zeroed bytes
struct BitWriter {
    uint8_t* p;
    uint64_t acc;
    int n;
    __device__ void put(uint32_t v, int bits) {
        acc |= (uint64_t)v << n;
        n += bits;
        while (n >= 8) {
            *p++ = (uint8_t)acc;
            acc >>= 8;
            n -= 8;
        }
    }
    __device__ void flush() {
        if (n > 0) *p++ = (uint8_t)acc;
        acc = 0;
        n = 0;
    }
};

// rec_off: absolute byte offset of each record in out (records of channel c
// follow channel c-1's).
__global__ void k_enc_records(const uint8_t* __restrict__ desc, const uint16_t* __restrict__ zv, int64_t nrec, int M,
                              int bsq, const uint64_t* __restrict__ rec_off, uint8_t* __restrict__ out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrec) return;
    uint8_t* rec = out + rec_off[r];
    const int nbm = (M + 7) >> 3;
    for (int i = 0; i < nbm; ++i) rec[i] = 0;
    uint8_t* cur = rec + nbm;
    const uint8_t* d = desc + r * M;
    for (int n = 0; n < M; ++n) {
        const int dd = d[n];
        if (dd == 0xFF) continue;
        rec[n >> 3] |= (uint8_t)(1u << (n & 7));
        *cur++ = (uint8_t)dd;
        const uint16_t* z = zv + (r * M + n) * bsq;
        const int mode = desc_mode(dd), bits = desc_bits(dd);
        BitWriter w{cur, 0, 0};
        if (mode == MODE_BITS) {
            for (int k = 0; k < bsq; ++k) w.put(z[k], bits);
        } else {
            // kernels.py:92-125: per group of <= 5 (trit) / 3 (quint) values
            // a base-3 / base-5 pack of the high digits, then the low fields
            const int group = mode == MODE_TRIT ? 5 : 3, radix = mode == MODE_TRIT ? 3 : 5,
                      pbits = mode == MODE_TRIT ? 8 : 7;
            const uint32_t mask = (1u << bits) - 1u;
            for (int g0 = 0; g0 < bsq; g0 += group) {
                const int gn = min(group, bsq - g0);
                uint32_t pack = 0, mul = 1;
                for (int i = 0; i < gn; ++i) {
                    pack += ((uint32_t)z[g0 + i] >> bits) * mul;
                    mul *= radix;
                }
                w.put(pack, pbits);
                if (bits > 0)
                    for (int i = 0; i < gn; ++i) w.put(z[g0 + i] & mask, bits);
            }
        }
        w.flush();
        cur += payload_bytes(dd, bsq);
    }
}

}  // namespace enc
}  // namespace rlfc

using namespace rlfc;

static int enc_status() { return cudaGetLastError() == cudaSuccess ? RLFC_OK : RLFC_ERR_CUDA; }

extern "C" int rlfc_enc_planes(const uint8_t* rgb, int64_t nimg, int32_t W, int32_t h_valid, int32_t hp, int32_t wp,
                               int32_t* planes, void* stream) {
    if (!rgb && h_valid > 0) return RLFC_ERR_ARGUMENT;
    if (!planes || nimg < 0 || W < 1 || hp < 1 || wp < W) return RLFC_ERR_ARGUMENT;
    enc::k_enc_planes<<<2048, 256, 0, static_cast<cudaStream_t>(stream)>>>(rgb, nimg, W, h_valid, hp, wp, planes);
    return enc_status();
}

extern "C" int rlfc_enc_pyramid(const int32_t* child, int32_t sx, int32_t sy, int32_t* parent, int32_t px, int32_t py,
                                const int64_t* weights, int32_t hp, int32_t wp, void* stream) {
    if (!child || !parent || !weights || sx < 1 || sy < 1 || px < 1 || py < 1) return RLFC_ERR_ARGUMENT;
    enc::k_enc_pyramid<<<2048, 256, 0, static_cast<cudaStream_t>(stream)>>>(child, sx, sy, parent, px, py, weights,
                                                                           (int64_t)hp * wp);
    return enc_status();
}

extern "C" int rlfc_enc_srv_level(int32_t* planes, const int32_t* above, int32_t sx, int32_t sy, int32_t psy,
                                  int32_t hp, int32_t wp, int32_t block, int32_t pixel_threshold,
                                  int64_t block_threshold, int32_t shift, int32_t level_base, int32_t m_nodes,
                                  uint8_t* desc, uint16_t* zv, uint64_t* present, int32_t* err, void* stream) {
    if (!planes || !above || !desc || !zv || !present || !err || hp % block || wp % block) return RLFC_ERR_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto pr = reinterpret_cast<unsigned long long*>(present);
#define RLFC_ENC(BB)                                                                                              \
    enc::k_enc_srv<BB><<<4096, 256, 0, s>>>(planes, above, sx, sy, psy, hp, wp, pixel_threshold, block_threshold, \
                                           shift, level_base, m_nodes, desc, zv, pr, err)
    switch (block) {
        case 2: RLFC_ENC(2); break;
        case 4: RLFC_ENC(4); break;
        case 8: RLFC_ENC(8); break;
        case 16: RLFC_ENC(16); break;
        default: return RLFC_ERR_ARGUMENT;
    }
#undef RLFC_ENC
    return enc_status();
}

extern "C" int rlfc_enc_record_sizes(const uint8_t* desc, int64_t nrec, int32_t m_nodes, int32_t bsq, uint64_t* size,
                                     void* stream) {
    if (!desc || !size || nrec < 0 || m_nodes < 1) return RLFC_ERR_ARGUMENT;
    if (nrec == 0) return RLFC_OK;
    enc::k_enc_rec_size<<<(unsigned)((nrec + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        desc, nrec, m_nodes, bsq, size);
    return enc_status();
}

extern "C" int rlfc_enc_records(const uint8_t* desc, const uint16_t* zv, int64_t nrec, int32_t m_nodes, int32_t bsq,
                                const uint64_t* rec_off, uint8_t* out, void* stream) {
    if (!desc || !zv || !rec_off || !out || nrec < 0 || m_nodes < 1) return RLFC_ERR_ARGUMENT;
    if (nrec == 0) return RLFC_OK;
    enc::k_enc_records<<<(unsigned)((nrec + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        desc, zv, nrec, m_nodes, bsq, rec_off, out);
    return enc_status();
}
