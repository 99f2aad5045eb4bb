// rlfc_kernels_abi.cu -- the reference's kernel-module signatures on the GPU
// (INTEGRATION.md Route 2: a drop-in for rlfc.kernels).
//
// The reference's decoder calls decode_chain_core / decode_plane_core
// (kernels.py:162-242) with an explicit ascending target list (the image's
// ancestor chain, decoder.py:101-104, 179-182) instead of image coordinates.
// These kernels take exactly those arguments: the SRV bytes, record offsets
// and targets, and walk each record like the reference (absent targets
// contribute 0; early exit after the last target; code 1 on a corrupt pack,
// 2 on a bad descriptor).  Reads stay inside the SRV section: a descriptor
// or payload past its end reports 2 (the reference has no bounds checks).
#include <cuda_runtime.h>
#include <atomic>
#include <climits>
#include <cstdint>

#include "rlfc_common.cuh"

namespace rlfc {
namespace kabi {

__device__ const DigitLut g_lut = make_digit_lut();

// kernels.py:162-216 with an explicit target list; acc (bsq values) holds
// the pre-filled root block and receives the dequantised target residuals.
__device__ int walk_targets(const uint8_t* srv, uint64_t srv_len, uint64_t rec_off, int m_nodes, int bsq,
                            const int64_t* targets, int nt, int shift, int32_t* acc) {
    if (nt == 0) return 0;
    const uint64_t bm = (uint64_t)(m_nodes + 7) >> 3;
    if (rec_off + bm > srv_len) return 2;
    const uint8_t* rec = srv + rec_off;
    uint64_t cursor = rec_off + bm;
    const int64_t last = targets[nt - 1];
    int ti = 0;
    for (int node = 0; node < m_nodes; ++node) {
        if (node > last) break;
        const int present = (rec[node >> 3] >> (node & 7)) & 1;
        if (!present) {
            if (ti < nt && targets[ti] == node && ++ti == nt) return 0;
            continue;
        }
        if (cursor >= srv_len) return 2;
        const int desc = srv[cursor];
        if (desc >= NUM_DESC) return 2;
        const uint64_t pbytes = (uint64_t)payload_bytes(desc, bsq);
        if (cursor + 1 + pbytes > srv_len) return 2;
        if (ti < nt && targets[ti] == node) {
            int32_t v[256];
            for (int j = 0; j < bsq; ++j) v[j] = 0;
            int st = 0;
            switch (bsq) {
                case 4: st = decode_payload_acc<4, true>(srv + cursor + 1, desc, shift, v, g_lut); break;
                case 16: st = decode_payload_acc<16, true>(srv + cursor + 1, desc, shift, v, g_lut); break;
                case 64: st = decode_payload_acc<64, true>(srv + cursor + 1, desc, shift, v, g_lut); break;
                default: st = decode_payload_acc<256, true>(srv + cursor + 1, desc, shift, v, g_lut); break;
            }
            if (st) return st;
            for (int j = 0; j < bsq; ++j) acc[j] += v[j];
            if (++ti == nt) return 0;
        }
        cursor += 1 + pbytes;
    }
    return 0;
}

// One thread per record: out[i*bsq ..] in/out, status[i].
__global__ void k_chain_core(const uint8_t* srv, uint64_t srv_len, const uint64_t* rec_offs, int n, int m_nodes,
                             int bsq, const int64_t* targets, int nt, int shift, int32_t* out, int32_t* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t acc[256];
    for (int j = 0; j < bsq; ++j) acc[j] = out[(int64_t)i * bsq + j];
    const int st = walk_targets(srv, srv_len, rec_offs[i], m_nodes, bsq, targets, nt, shift, acc);
    status[i] = st;
    for (int j = 0; j < bsq; ++j) out[(int64_t)i * bsq + j] = acc[j];
}

// One request, latency path: the targets ride in the kernel parameters and
// the block lives in the caller's pinned host buffer (io[0..bsq) = the root
// block in, the result out), status word io[bsq] written last.
struct ChainOne {
    int64_t targets[16];
};

__global__ void k_chain_core_one(const uint8_t* srv, uint64_t srv_len, uint64_t rec_off, int m_nodes, int bsq,
                                 const __grid_constant__ ChainOne tg, int nt, int shift, volatile int32_t* io) {
    int32_t acc[256];
    for (int j = 0; j < bsq; ++j) acc[j] = io[j];
    const int st = walk_targets(srv, srv_len, rec_off, m_nodes, bsq, tg.targets, nt, shift, acc);
    for (int j = 0; j < bsq; ++j) io[j] = acc[j];
    __threadfence_system();
    io[bsq] = st;
}

// kernels.py:219-242: every block of one plane; the failure word keeps the
// first failing block in row-major order (the reference returns there).
__global__ void k_plane_core(const uint8_t* srv, uint64_t srv_len, const uint64_t* offsets, int bxn, int byn,
                             int m_nodes, int block, const int64_t* targets, int nt, int shift,
                             const int32_t* root_plane, int32_t* out_plane, unsigned long long* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= bxn * byn) return;
    const int by = i / bxn, bx = i - by * bxn, bsq = block * block, wp = bxn * block;
    int32_t acc[256];
    for (int yy = 0; yy < block; ++yy)
        for (int xx = 0; xx < block; ++xx)
            acc[yy * block + xx] = root_plane[(int64_t)(by * block + yy) * wp + bx * block + xx];
    const int st = walk_targets(srv, srv_len, offsets[i], m_nodes, bsq, targets, nt, shift, acc);
    if (st) {
        atomicMin(status, (unsigned long long)i << 2 | (unsigned long long)st);
        return;
    }
    for (int yy = 0; yy < block; ++yy)
        for (int xx = 0; xx < block; ++xx)
            out_plane[(int64_t)(by * block + yy) * wp + bx * block + xx] = acc[yy * block + xx];
}

}  // namespace kabi
}  // namespace rlfc

using namespace rlfc;

extern "C" int rlfc_chain_core(const uint8_t* srv, uint64_t srv_len, const uint64_t* rec_offs, int32_t n,
                               int32_t m_nodes, int32_t bsq, const int64_t* targets, int32_t nt, int32_t shift,
                               int32_t* out, int32_t* status, void* stream) {
    if (!srv || !rec_offs || !out || !status || n < 0 || nt < 0 || (nt && !targets) || m_nodes < 1 ||
        (bsq != 4 && bsq != 16 && bsq != 64 && bsq != 256) || shift < 0 || shift > 30)
        return RLFC_ERR_ARGUMENT;
    if (n == 0) return RLFC_OK;
    kabi::k_chain_core<<<(n + 63) / 64, 64, 0, static_cast<cudaStream_t>(stream)>>>(
        srv, srv_len, rec_offs, n, m_nodes, bsq, targets, nt, shift, out, status);
    return cudaGetLastError() == cudaSuccess ? RLFC_OK : RLFC_ERR_CUDA;
}

extern "C" int rlfc_plane_core(const uint8_t* srv, uint64_t srv_len, const uint64_t* offsets, int32_t blocks_x,
                               int32_t blocks_y, int32_t m_nodes, int32_t block, const int64_t* targets, int32_t nt,
                               int32_t shift, const int32_t* root_plane, int32_t* out_plane, uint64_t* status,
                               void* stream) {
    if (!srv || !offsets || !root_plane || !out_plane || !status || blocks_x < 1 || blocks_y < 1 || nt < 0 ||
        (nt && !targets) || m_nodes < 1 || (block != 2 && block != 4 && block != 8 && block != 16) || shift < 0 ||
        shift > 30)
        return RLFC_ERR_ARGUMENT;
    const int n = blocks_x * blocks_y;
    kabi::k_plane_core<<<(n + 63) / 64, 64, 0, static_cast<cudaStream_t>(stream)>>>(
        srv, srv_len, offsets, blocks_x, blocks_y, m_nodes, block, targets, nt, shift, root_plane, out_plane,
        reinterpret_cast<unsigned long long*>(status));
    return cudaGetLastError() == cudaSuccess ? RLFC_OK : RLFC_ERR_CUDA;
}

extern "C" int rlfc_chain_core_sync(const uint8_t* srv, uint64_t srv_len, uint64_t rec_off, int32_t m_nodes,
                                    int32_t bsq, const int64_t* targets, int32_t nt, int32_t shift, int32_t* io,
                                    void* stream) {
    if (!srv || !io || nt < 0 || nt > 16 || (nt && !targets) || m_nodes < 1 ||
        (bsq != 4 && bsq != 16 && bsq != 64 && bsq != 256) || shift < 0 || shift > 30)
        return RLFC_ERR_ARGUMENT;
    kabi::ChainOne tg{};
    for (int i = 0; i < nt; ++i) tg.targets[i] = targets[i];
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    volatile int32_t* flag = io + bsq;
    *flag = INT_MIN;                           // never a status value
    std::atomic_thread_fence(std::memory_order_seq_cst);
    kabi::k_chain_core_one<<<1, 1, 0, st>>>(srv, srv_len, rec_off, m_nodes, bsq, tg, nt, shift, io);
    if (cudaGetLastError() != cudaSuccess) return RLFC_ERR_CUDA;
    // poll the status word (a stream synchronize's wake-up is most of one
    // request's latency); query the stream every 1024 polls so a failed
    // launch cannot hang the caller
    for (uint32_t i = 1; *flag == INT_MIN; ++i) {
        if ((i & 1023u) == 0) {
            const cudaError_t q = cudaStreamQuery(st);
            if (q == cudaErrorNotReady) continue;
            if (q != cudaSuccess) return RLFC_ERR_CUDA;
            if (*flag == INT_MIN) return RLFC_ERR_CUDA;
            break;
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return RLFC_OK;
}
