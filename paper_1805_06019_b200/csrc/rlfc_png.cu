// rlfc_png.cu -- root-view decode at init: PNG unfiltering on the GPU.
//
// The reference decodes each 16-bit greyscale root plane with Pillow
// (container.py:175-195) as part of init (decoder.py:31-48); on cfg2 that is
// most of init.  The host here only inflates the IDAT zlib stream (threads);
// the scanline filters (PNG spec: None / Sub / Up / Average / Paeth, bytes
// per pixel 2) are undone on the GPU.  Every output byte depends on its left
// neighbour (same byte lane, 2 bytes back) and on the row above, so a CTA of
// up to 1024 threads runs one plane as a wavefront: thread r owns row r and
// processes sample j at step r + j, taking the row above from thread r-1
// through a small shared-memory ring.  Rows beyond 1024 run in further
// passes that read their row above from the output.  Samples are big-endian
// (PNG); k_root_planes then removes the channel bias (container.py:56) into
// the device root tensor layout.
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/rlfc_b200.h"

namespace rlfc {
namespace png {

constexpr int MAXT = 1024;

__device__ __forceinline__ uint32_t paeth(uint32_t a, uint32_t b, uint32_t c) {
    const int p = (int)a + (int)b - (int)c;
    const int pa = abs(p - (int)a), pb = abs(p - (int)b), pc = abs(p - (int)c);
    return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

// One byte: filter f, raw byte x, left a, up b, up-left c (PNG 9.2-9.4).
__device__ __forceinline__ uint32_t unf(int f, uint32_t x, uint32_t a, uint32_t b, uint32_t c) {
    switch (f) {
        case 0: return x;
        case 1: return (x + a) & 255u;
        case 2: return (x + b) & 255u;
        case 3: return (x + ((a + b) >> 1)) & 255u;
        default: return (x + paeth(a, b, c)) & 255u;
    }
}

// raw: per plane, height rows of (1 + 2*width) filtered bytes; out: per plane
// height x width uint16 sample values.  bad: set on a filter type > 4.
__global__ void __launch_bounds__(MAXT) k_unfilter(const uint8_t* raw, int64_t raw_plane, int width, int height,
                                                   uint16_t* out, int64_t out_plane, int* bad) {
    __shared__ uint16_t ring[MAXT][4];           // sample j of row r at ring[r][j & 3]
    const int r0 = threadIdx.x;
    const uint8_t* rp = raw + (int64_t)blockIdx.x * raw_plane;
    uint16_t* op = out + (int64_t)blockIdx.x * out_plane;
    const int stride = 1 + 2 * width;
    for (int base = 0; base < height; base += blockDim.x) {
        const int r = base + r0;
        const bool live = r < height;
        const int nrows = min((int)blockDim.x, height - base);
        const uint8_t* row = rp + (int64_t)(live ? r : 0) * stride;
        const int f = live ? row[0] : 0;
        if (live && f > 4) atomicExch(bad, 1);
        const uint16_t* above = r > 0 && r0 == 0 ? op + (int64_t)(r - 1) * width : nullptr;  // previous pass
        uint32_t a_hi = 0, a_lo = 0, c_hi = 0, c_lo = 0;      // left / up-left bytes
        for (int d = 0; d < width + nrows - 1; ++d) {
            const int j = d - r0;
            uint32_t v = 0;
            const bool act = live && j >= 0 && j < width;
            if (act) {
                uint32_t up = 0;
                if (r > 0) up = r0 > 0 ? ring[r0 - 1][j & 3] : above[j];
                const uint32_t b_hi = up >> 8, b_lo = up & 255u;
                const uint32_t x_hi = row[1 + 2 * j], x_lo = row[2 + 2 * j];
                const uint32_t hi = unf(f, x_hi, a_hi, b_hi, c_hi), lo = unf(f, x_lo, a_lo, b_lo, c_lo);
                a_hi = hi;
                a_lo = lo;
                c_hi = b_hi;
                c_lo = b_lo;
                v = hi << 8 | lo;
                op[(int64_t)r * width + j] = (uint16_t)v;
            }
            __syncthreads();                      // the row above's sample j - 1 is read next step
            if (act) ring[r0][j & 3] = (uint16_t)v;
            __syncthreads();
        }
        __syncthreads();
    }
}

// Root tensor (rsx, rsy, 3, hp, wp): sample - bias (0, 256, 256), as int16
// when i16 (the caller checked the range) else int32; plane p of the decode
// order (c outer, y, x inner: container.py:355-379) goes to root (x, y, c).
__global__ void k_root_planes(const uint16_t* in, int nplanes, int rsx, int rsy, int hp, int wp, int i16, void* dst,
                              int* minmax) {
    const int64_t pl = (int64_t)hp * wp;
    const int64_t n = pl * nplanes;
    int lo = 1 << 30, hi = -(1 << 30);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)(i / pl);
        const int64_t o = i - (int64_t)p * pl;
        const int c = p / (rsx * rsy), yx = p % (rsx * rsy), y = yx / rsx, x = yx % rsx;
        const int v = (int)in[i] - (c ? 256 : 0);
        const int64_t d = (((int64_t)x * rsy + y) * 3 + c) * pl + o;
        if (i16) static_cast<int16_t*>(dst)[d] = (int16_t)v;
        else static_cast<int32_t*>(dst)[d] = v;
        lo = min(lo, v);
        hi = max(hi, v);
    }
    if (minmax) {
        atomicMin(minmax, lo);
        atomicMax(minmax + 1, hi);
    }
}

}  // namespace png
}  // namespace rlfc

using namespace rlfc;

extern "C" int rlfc_png_unfilter(const uint8_t* raw, int64_t raw_plane, int32_t nplanes, int32_t width,
                                 int32_t height, uint16_t* out, int64_t out_plane, int32_t* bad, void* stream) {
    if (!raw || !out || !bad || nplanes < 0 || width < 1 || height < 1) return RLFC_ERR_ARGUMENT;
    if (raw_plane < (int64_t)height * (1 + 2 * (int64_t)width) || out_plane < (int64_t)height * width)
        return RLFC_ERR_ARGUMENT;
    if (nplanes == 0) return RLFC_OK;
    const int threads = height < png::MAXT ? height : png::MAXT;
    png::k_unfilter<<<nplanes, threads, 0, static_cast<cudaStream_t>(stream)>>>(raw, raw_plane, width, height, out,
                                                                                 out_plane, bad);
    return cudaGetLastError() == cudaSuccess ? RLFC_OK : RLFC_ERR_CUDA;
}

extern "C" int rlfc_root_planes(const uint16_t* samples, int32_t nplanes, int32_t rsx, int32_t rsy, int32_t hp,
                                int32_t wp, int32_t i16, void* dst, int32_t* minmax, void* stream) {
    if (!samples || !dst || nplanes != 3 * rsx * rsy || hp < 1 || wp < 1) return RLFC_ERR_ARGUMENT;
    png::k_root_planes<<<592, 256, 0, static_cast<cudaStream_t>(stream)>>>(samples, nplanes, rsx, rsy, hp, wp, i16,
                                                                          dst, minmax);
    return cudaGetLastError() == cudaSuccess ? RLFC_OK : RLFC_ERR_CUDA;
}
