// rlfc_render.cu -- novel-view rendering over decoded camera images.
//
// Bit-exact restatement of the reference renderer's float64 arithmetic
// (/root/reference/pkg/src/rlfc/renderer.py).  Every multiply / add / divide
// is an explicit round-to-nearest intrinsic (__dmul_rn, __dadd_rn,
// __ddiv_rn), so nvcc can never contract a*b+c into an FMA -- numpy does not
// either -- and the operation order is numpy's.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/rlfc_b200.h"
#include "rlfc_field.cuh"

namespace rlfc {

constexpr double SNAP_EPS = 1e-9;  // renderer.py:23

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dadd_rn(a, -b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// renderer.py:82-84 _snap (Python round() is half-to-even = rint)
__device__ __forceinline__ double snap(double f) {
    double r = rint(f);
    return fabs(sub(f, r)) < SNAP_EPS ? r : f;
}

// renderer.py:119-131 _axis_taps: clamp, split, drop zero-weight taps.
__device__ __forceinline__ int axis_taps(double coord, int count, int* idx, double* w) {
    double c = fmin(fmax(coord, 0.0), (double)(count - 1));
    if (count == 1) {
        idx[0] = 0;
        w[0] = 1.0;
        return 1;
    }
    int i0 = min((int)floor(c), count - 2);
    double f = snap(sub(c, (double)i0));
    int n = 0;
    if (f < 1.0) { idx[n] = i0; w[n] = sub(1.0, f); ++n; }
    if (f > 0.0) { idx[n] = i0 + 1; w[n] = f; ++n; }
    return n;
}

// renderer.py:221-230 _vec_taps (keeps zero-weight taps).
__device__ __forceinline__ void vec_tap(double coord, int count, int& i0, double& f) {
    double c = fmin(fmax(coord, 0.0), (double)(count - 1));
    if (count == 1) { i0 = 0; f = 0.0; return; }
    double fl = fmin(floor(c), (double)(count - 2));
    i0 = (int)fl;
    double fr = sub(c, (double)i0);
    double r = rint(fr);
    f = fabs(sub(fr, r)) < SNAP_EPS ? r : fr;
}

// np.interp(x, arange(n), arange(n)) on the identity camera grid
// (renderer.py:75-79, 177-178): x clamped to [0, n-1], exact inside.
__device__ __forceinline__ double interp_identity(double x, int n) {
    return x < 0.0 ? 0.0 : (x > (double)(n - 1) ? (double)(n - 1) : x);
}

__device__ __forceinline__ uint8_t round_clip(double a) {
    double fl = floor(add(a, 0.5));  // renderer.py:274 floor(acc + 0.5).clip(0, 255)
    return fl < 0.0 ? 0 : (fl > 255.0 ? 255 : (uint8_t)fl);
}

// Slab poses (renderer.py:233-276).  A ray's image-plane hit, hence its u
// tap, depends only on the output column, and its v tap only on the row
// (the eye and the focal plane are per pose), so one CTA per (pose, band of
// RB output rows) evaluates the column and row terms once into shared memory
// with exactly the reference's operations, and each pixel then only blends
// its 16 taps in the reference's (s, t, p, q) order.
constexpr int RB = 16;
struct AxisTap {
    double f;      // fraction of the upper tap
    int i0;        // lower tap index
    int inside;    // hit within the image-plane window along this axis
};

// renderer.py:177-187 + 251-261 along one axis: target, direction, hit,
// window test, texel coordinate, snap, _vec_taps.
__device__ __forceinline__ AxisTap slab_axis(int i, int n_out, double lo, double hi, double e, double tp, int n_px) {
    const double wdt = sub(hi, lo);
    const double tx = add(lo, dvd(mul(add((double)i, 0.5), wdt), (double)n_out));
    const double dx = sub(tx, e);
    const double ix = add(e, mul(tp, dx));
    AxisTap a;
    a.inside = lo <= ix && ix <= hi;
    double u = sub(mul(dvd(sub(ix, lo), wdt), (double)n_px), 0.5);
    const double ru = rint(u);
    if (fabs(sub(u, ru)) < SNAP_EPS) u = ru;
    vec_tap(u, n_px, a.i0, a.f);
    return a;
}

__global__ void __launch_bounds__(256) k_render_slab(const uint8_t* __restrict__ field,
                                                     const int32_t* __restrict__ slots, int S, int T, int W, int H,
                                                     const double* __restrict__ poses,
                                                     const rlfc_render_geom* __restrict__ geoms,
                                                     const uint8_t* __restrict__ bgs, int ow, int oh,
                                                     uint8_t* __restrict__ out, int rb) {
    extern __shared__ __align__(16) uint8_t rsm[];
    AxisTap* cols = reinterpret_cast<AxisTap*>(rsm);          // [ow]
    AxisTap* rows = cols + ow;                                 // [rb]
    const int v = blockIdx.y;
    const int j0 = blockIdx.x * rb;
    const int nrow = min(rb, oh - j0);
    const rlfc_render_geom g = geoms[v];
    const double ps = poses[4 * v], pt = poses[4 * v + 1];
    const double focal = poses[4 * v + 2] != 0.0 ? poses[4 * v + 3] : g.img_z;
    const double ex = interp_identity(ps, S), ey = interp_identity(pt, T), ez = g.cam_z;
    const double dz = sub(focal, ez);
    const double tp = dvd(sub(g.img_z, ez), dz);
    for (int i = threadIdx.x; i < ow + nrow; i += blockDim.x) {
        if (i < ow) cols[i] = slab_axis(i, ow, g.x0, g.x1, ex, tp, W);
        else rows[i - ow] = slab_axis(j0 + i - ow, oh, g.y0, g.y1, ey, tp, H);
    }
    // renderer.py:265-266 camera taps (per pose)
    int si[2], ti[2];
    double ws[2], wt[2];
    const int ns = axis_taps(snap(ex), S, si, ws);
    const int nt = axis_taps(snap(ey), T, ti, wt);
    const int64_t img = (int64_t)W * H * 3;
    const uint8_t* ims[4];
    double wst[4];
    int nab = 0;
    for (int a = 0; a < ns; ++a)
        for (int b = 0; b < nt; ++b) {
            const int cam = si[a] * T + ti[b];
            ims[nab] = field + (int64_t)(slots ? slots[cam] : cam) * img;
            wst[nab] = mul(ws[a], wt[b]);
            ++nab;
        }
    __syncthreads();
    const uint8_t* bg = bgs + 3 * v;
    for (int q = threadIdx.x; q < nrow * ow; q += blockDim.x) {
        const int jr = q / ow, i = q - jr * ow;
        const AxisTap cu = cols[i], cv = rows[jr];
        uint8_t* o = out + (((int64_t)v * oh + j0 + jr) * ow + i) * 3;
        if (!(cu.inside && cv.inside)) {
            o[0] = bg[0]; o[1] = bg[1]; o[2] = bg[2];
            continue;
        }
        const int gx0 = min(cu.i0, W - 1), gx1 = min(cu.i0 + 1, W - 1);
        const int gy0 = min(cv.i0, H - 1), gy1 = min(cv.i0 + 1, H - 1);
        const double wu[2] = {sub(1.0, cu.f), cu.f}, wv[2] = {sub(1.0, cv.f), cv.f};
        const int gx[2] = {gx0, gx1}, gy[2] = {gy0, gy1};
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
        for (int ab = 0; ab < nab; ++ab) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const double wsu = mul(wst[ab], wu[p]);
#pragma unroll
                for (int qq = 0; qq < 2; ++qq) {
                    const double w = mul(wsu, wv[qq]);
                    const uint8_t* px = ims[ab] + ((int64_t)gy[qq] * W + gx[p]) * 3;
                    acc0 = add(acc0, mul(w, (double)px[0]));
                    acc1 = add(acc1, mul(w, (double)px[1]));
                    acc2 = add(acc2, mul(w, (double)px[2]));
                }
            }
        }
        o[0] = round_clip(acc0);
        o[1] = round_clip(acc1);
        o[2] = round_clip(acc2);
    }
}

struct PinholeCoord {
    bool hit;
    double s, t, u, v;
};

// renderer.py:190-209 per-pixel direction + renderer.py:87-116
// ray_to_lf_coords.  parallel is set when |dir.z| < 1e-15.
__device__ __forceinline__ PinholeCoord pinhole_coord(const double* fr, const rlfc_render_geom& g, int S, int T,
                                                      int W, int H, int i, int j, int ow, int oh, bool& parallel) {
    PinholeCoord c{false, 0, 0, 0, 0};
    const double half = fr[12], aspect = fr[13];
    const double px = sub(mul(dvd(add((double)i, 0.5), (double)ow), 2.0), 1.0);
    const double py = sub(mul(dvd(add((double)j, 0.5), (double)oh), 2.0), 1.0);
    const double a = mul(mul(px, half), aspect), b = mul(py, half);
    double d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = add(add(fr[3 + k], mul(a, fr[6 + k])), mul(b, fr[9 + k]));
    if (fabs(d[2]) < 1e-15) {
        parallel = true;
        return c;
    }
    const double tc = dvd(sub(g.cam_z, fr[2]), d[2]);
    const double cx = add(fr[0], mul(tc, d[0])), cy = add(fr[1], mul(tc, d[1]));
    if (!(0.0 <= cx && cx <= (double)(S - 1) && 0.0 <= cy && cy <= (double)(T - 1))) return c;
    const double tt = dvd(sub(g.img_z, fr[2]), d[2]);
    const double ix = add(fr[0], mul(tt, d[0])), iy = add(fr[1], mul(tt, d[1]));
    if (!(g.x0 <= ix && ix <= g.x1 && g.y0 <= iy && iy <= g.y1)) return c;
    c.hit = true;
    c.s = snap(interp_identity(cx, S));
    c.t = snap(interp_identity(cy, T));
    c.u = snap(sub(mul(dvd(sub(ix, g.x0), sub(g.x1, g.x0)), (double)W), 0.5));
    c.v = snap(sub(mul(dvd(sub(iy, g.y0), sub(g.y1, g.y0)), (double)H), 0.5));
    return c;
}

// One thread per output pixel of one pinhole pose (renderer.py:295-305 +
// sample_quadrilinear renderer.py:147-169).
__global__ void k_render_pinhole(const uint8_t* __restrict__ field, const int32_t* __restrict__ slots, int S, int T,
                                 int W, int H,
                                 const double* __restrict__ frames, const rlfc_render_geom* __restrict__ geoms,
                                 const uint8_t* __restrict__ bgs, int ow, int oh, uint8_t* __restrict__ out,
                                 int32_t* status) {
    const int v = blockIdx.y;
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= (int64_t)ow * oh) return;
    const int i = (int)(pix % ow), j = (int)(pix / ow);
    uint8_t* o = out + ((int64_t)v * oh * ow + pix) * 3;
    const uint8_t* bg = bgs + 3 * v;
    bool parallel = false;
    PinholeCoord c = pinhole_coord(frames + 14 * v, geoms[v], S, T, W, H, i, j, ow, oh, parallel);
    if (parallel) atomicExch(status + v, -2);
    if (!c.hit) {
        o[0] = bg[0]; o[1] = bg[1]; o[2] = bg[2];
        return;
    }
    int si[2], ti[2], ui[2], vi[2];
    double ws[2], wt[2], wu[2], wv[2];
    const int ns = axis_taps(c.s, S, si, ws), nt = axis_taps(c.t, T, ti, wt);
    const int nu = axis_taps(c.u, W, ui, wu), nv = axis_taps(c.v, H, vi, wv);
    const int64_t img = (int64_t)W * H * 3;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int a = 0; a < ns; ++a)
        for (int b = 0; b < nt; ++b)
            for (int p = 0; p < nu; ++p)
                for (int q = 0; q < nv; ++q) {
                    const double w = mul(mul(mul(ws[a], wt[b]), wu[p]), wv[q]);
                    const int cam = si[a] * T + ti[b];
                    const uint8_t* px = field + (int64_t)(slots ? slots[cam] : cam) * img +
                                        ((int64_t)vi[q] * W + ui[p]) * 3;
                    acc0 = add(acc0, mul(w, (double)px[0]));
                    acc1 = add(acc1, mul(w, (double)px[1]));
                    acc2 = add(acc2, mul(w, (double)px[2]));
                }
    o[0] = round_clip(acc0);
    o[1] = round_clip(acc1);
    o[2] = round_clip(acc2);
}

__global__ void k_pinhole_needs(int S, int T, int W, int H, const double* __restrict__ frames,
                                const rlfc_render_geom* __restrict__ geoms, int ow, int oh,
                                uint8_t* __restrict__ need) {
    const int v = blockIdx.y;
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= (int64_t)ow * oh) return;
    bool parallel = false;
    PinholeCoord c = pinhole_coord(frames + 14 * v, geoms[v], S, T, W, H, (int)(pix % ow), (int)(pix / ow), ow,
                                   oh, parallel);
    if (!c.hit) return;
    int si[2], ti[2];
    double ws[2], wt[2];
    const int ns = axis_taps(c.s, S, si, ws), nt = axis_taps(c.t, T, ti, wt);
    for (int a = 0; a < ns; ++a)
        for (int b = 0; b < nt; ++b) need[si[a] * T + ti[b]] = 1;
}

static int launch_status() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "rlfc_b200: CUDA launch error: %s\n", cudaGetErrorString(e));
        return RLFC_ERR_CUDA;
    }
    return RLFC_OK;
}

}  // namespace rlfc

using namespace rlfc;

extern "C" int rlfc_render_slab(const uint8_t* field, const int32_t* slots, int32_t S, int32_t T, int32_t W, int32_t H,
                                const double* poses, const rlfc_render_geom* geoms, const uint8_t* bg, int32_t n,
                                int32_t ow, int32_t oh, uint8_t* out, void* stream) {
    if (S < 1 || T < 1 || W < 1 || H < 1 || n < 0 || ow < 1 || oh < 1 || n > 65535) return RLFC_ERR_ARGUMENT;
    if (n == 0) return RLFC_OK;
    // rows per CTA: RB when the batch fills the GPU, fewer for small batches
    // (a single 512-row view is 32 CTAs at RB = 16: under a quarter of the SMs)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want_ctas = 4ll * sms;
    int rb = RB;
    while (rb > 1 && (int64_t)n * ((oh + rb - 1) / rb) < want_ctas) rb >>= 1;
    const size_t smem = (size_t)(ow + rb) * sizeof(AxisTap);
    if (smem > 200 * 1024) return RLFC_ERR_ARGUMENT;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_render_slab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)((oh + rb - 1) / rb), (unsigned)n);
    k_render_slab<<<grid, 256, smem, (cudaStream_t)stream>>>(field, slots, S, T, W, H, poses, geoms, bg, ow, oh, out,
                                                             rb);
    return launch_status();
}

extern "C" int rlfc_render_pinhole(const uint8_t* field, const int32_t* slots, int32_t S, int32_t T, int32_t W, int32_t H,
                                   const double* frames, const rlfc_render_geom* geoms, const uint8_t* bg,
                                   int32_t n, int32_t ow, int32_t oh, uint8_t* out, int32_t* status,
                                   void* stream) {
    if (S < 1 || T < 1 || W < 1 || H < 1 || n < 0 || ow < 1 || oh < 1 || n > 65535) return RLFC_ERR_ARGUMENT;
    if (n == 0) return RLFC_OK;
    const int threads = 256;
    dim3 grid((unsigned)(((int64_t)ow * oh + threads - 1) / threads), (unsigned)n);
    k_render_pinhole<<<grid, threads, 0, (cudaStream_t)stream>>>(field, slots, S, T, W, H, frames, geoms, bg, ow, oh, out,
                                                                 status);
    return launch_status();
}

extern "C" int rlfc_render_pinhole_needs(int32_t S, int32_t T, int32_t W, int32_t H, const double* frames,
                                         const rlfc_render_geom* geoms, int32_t n, int32_t ow, int32_t oh,
                                         uint8_t* need, void* stream) {
    if (S < 1 || T < 1 || W < 1 || H < 1 || n < 0 || ow < 1 || oh < 1 || n > 65535) return RLFC_ERR_ARGUMENT;
    if (n == 0) return RLFC_OK;
    const int threads = 256;
    dim3 grid((unsigned)(((int64_t)ow * oh + threads - 1) / threads), (unsigned)n);
    k_pinhole_needs<<<grid, threads, 0, (cudaStream_t)stream>>>(S, T, W, H, frames, geoms, ow, oh, need);
    return launch_status();
}

// ---- one call per batch of slab poses (host runtime) ------------------------------------
// renderer.render_views for SlabPose batches without Python in the loop: the
// tap-camera set (floor and ceil of each clamped eye coordinate, a superset
// of renderer.py:119-131 _axis_taps), the slot table and camera rows are
// built here, staged with the poses, geometries and backgrounds in one
// pinned buffer and sent with one copy; the staged decode (slot mode) and
// k_render_slab follow on the same stream; the decode status word comes back
// with one small copy and the call returns after the stream has drained.
extern "C" int rlfc_render_slab_batch(const rlfc_field* f, int32_t stop_level, void* ws, uint64_t ws_bytes,
                                      uint64_t present, int32_t n_flagged, const double* poses,
                                      const rlfc_render_geom* geoms, const uint8_t* bg, int32_t n, int32_t ow,
                                      int32_t oh, uint8_t* field, int32_t field_cap, uint8_t* out,
                                      uint8_t* stage_host, uint8_t* stage_dev, uint64_t stage_bytes,
                                      uint8_t* out_host, uint64_t* status_word, void* stream) {
    if (!f || !poses || !geoms || !bg || !field || !out || !stage_host || !stage_dev || !status_word || n < 1 ||
        n > 65535 || ow < 1 || oh < 1)
        return RLFC_ERR_ARGUMENT;
    const int S = f->s_count, T = f->t_count, W = f->width, H = f->height;
    auto al = [](uint64_t x) { return (x + 15) & ~uint64_t(15); };
    const uint64_t o_stat = 0, o_pose = 16, o_geom = al(o_pose + 32ull * n), o_slot = al(o_geom + 48ull * n),
                   o_rows = al(o_slot + 4ull * S * T), o_bg = al(o_rows + 4ull * T), o_sel = al(o_bg + 3ull * n),
                   total = al(o_sel + 4ull * (1 + rlfc::SEL_NODES_MAX));
    if (total > stage_bytes) return RLFC_ERR_ARGUMENT;
    int32_t* slots = reinterpret_cast<int32_t*>(stage_host + o_slot);
    for (int i = 0; i < S * T; ++i) slots[i] = -1;
    auto cell = [](double x, int cnt, int hi) {
        const double c = fmin(fmax(x, 0.0), (double)(cnt - 1));
        return hi ? (int)ceil(c) : (int)floor(c);
    };
    for (int v = 0; v < n; ++v)
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) slots[cell(poses[4 * v], S, a) * T + cell(poses[4 * v + 1], T, b)] = 0;
    int ncam = 0, nrows = 0;
    int32_t* rows = reinterpret_cast<int32_t*>(stage_host + o_rows);
    for (int t = 0; t < T; ++t) {
        bool any = false;
        for (int s = 0; s < S; ++s)
            if (slots[s * T + t] == 0) any = true;
        if (any) rows[nrows++] = t;
    }
    int32_t views[4 * 64];
    int nviews = 0;
    for (int i = 0; i < S * T; ++i)
        if (slots[i] == 0) {
            if (nviews < 4 * 64) views[nviews] = i;
            ++nviews;
            slots[i] = ncam++;
        }
    if (ncam > field_cap) return RLFC_ERR_ARGUMENT;
    // the slot-mode node list, built here (no k_sel_nodes launch)
    uint32_t* sel = reinterpret_cast<uint32_t*>(stage_host + o_sel);
    const int sel_n = nviews <= 4 * 64 ? rlfc::sel_nodes_host(*f, stop_level, views, nviews, sel)
                                       : (int)(sel[0] = rlfc::SEL_NODES_MAX + 1);
    std::memset(stage_host + o_stat, 0, 16);
    std::memcpy(stage_host + o_pose, poses, 32ull * n);
    std::memcpy(stage_host + o_geom, geoms, 48ull * n);
    std::memcpy(stage_host + o_bg, bg, 3ull * n);
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemcpyAsync(stage_dev, stage_host, total, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return RLFC_ERR_CUDA;
    uint64_t* dstat = reinterpret_cast<uint64_t*>(stage_dev + o_stat);
    const int32_t* dslots = reinterpret_cast<const int32_t*>(stage_dev + o_slot);
    const int64_t img = (int64_t)H * W * 3;
    int rc = RLFC_ERR_ARGUMENT;
    if (ws)
        rc = rlfc::decode_field_staged_sel(f, stop_level, dslots, 0, f->hb, field, img, (int64_t)W * 3, ws, ws_bytes,
                                           present, n_flagged, reinterpret_cast<const int32_t*>(stage_dev + o_rows),
                                           nrows, dstat, stream, reinterpret_cast<const uint32_t*>(stage_dev + o_sel),
                                           sel_n);
    if (rc == RLFC_ERR_ARGUMENT)
        rc = rlfc_decode_field(f, stop_level, dslots, 0, f->hb, field, img, (int64_t)W * 3, dstat, stream);
    if (rc != RLFC_OK) return rc;
    rc = rlfc_render_slab(field, dslots, S, T, W, H, reinterpret_cast<const double*>(stage_dev + o_pose),
                          reinterpret_cast<const rlfc_render_geom*>(stage_dev + o_geom), stage_dev + o_bg, n, ow,
                          oh, out, stream);
    if (rc != RLFC_OK) return rc;
    if (out_host && cudaMemcpyAsync(out_host, out, (size_t)n * oh * ow * 3, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return RLFC_ERR_CUDA;
    if (cudaMemcpyAsync(stage_host + o_stat, dstat, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return RLFC_ERR_CUDA;
    std::memcpy(status_word, stage_host + o_stat, 8);
    return RLFC_OK;
}

extern "C" uint64_t rlfc_render_staging_bytes(const rlfc_field* f, int32_t n) {
    if (!f || n < 1) return 0;
    auto al = [](uint64_t x) { return (x + 15) & ~uint64_t(15); };
    const uint64_t o_geom = al(16 + 32ull * n), o_slot = al(o_geom + 48ull * n),
                   o_rows = al(o_slot + 4ull * f->s_count * f->t_count), o_bg = al(o_rows + 4ull * f->t_count),
                   o_sel = al(o_bg + 3ull * n);
    return al(o_sel + 4ull * (1 + rlfc::SEL_NODES_MAX));
}

// ---- one image in one call (host runtime) ----------------------------------------------
// decoder.decode_image (decoder.py:187-194) without Python in the loop: the
// slot table (one view) and its camera row are staged with the status word
// in one pinned buffer and sent with one copy; the staged decode in slot mode
// (else the fused decode) fills rgb_dev, the image and the status come back
// with two copies on the same stream, and the call returns after it drained.
extern "C" int rlfc_decode_image_host(const rlfc_field* f, int32_t stop_level, void* ws, uint64_t ws_bytes,
                                      uint64_t present, int32_t n_flagged, int32_t s, int32_t t, uint8_t* rgb_dev,
                                      uint8_t* rgb_host, uint8_t* stage_host, uint8_t* stage_dev,
                                      uint64_t stage_bytes, uint64_t* status_word, void* stream) {
    if (!f || !rgb_dev || !rgb_host || !stage_host || !stage_dev || !status_word) return RLFC_ERR_ARGUMENT;
    const int S = f->s_count, T = f->t_count, W = f->width, H = f->height;
    if (s < 0 || s >= S || t < 0 || t >= T || stop_level < 0 || stop_level > f->tree_height) return RLFC_ERR_ARGUMENT;
    const uint64_t o_slot = 16, o_rows = (o_slot + 4ull * S * T + 15) & ~15ull, o_sel = o_rows + 16,
                   total = o_sel + 4ull * (1 + rlfc::SEL_NODES_MAX);
    if (total > stage_bytes) return RLFC_ERR_ARGUMENT;
    std::memset(stage_host, 0, 16);
    int32_t* slots = reinterpret_cast<int32_t*>(stage_host + o_slot);
    for (int i = 0; i < S * T; ++i) slots[i] = -1;
    slots[s * T + t] = 0;
    reinterpret_cast<int32_t*>(stage_host + o_rows)[0] = t;
    const int32_t view = s * T + t;
    const int sel_n = rlfc::sel_nodes_host(*f, stop_level, &view, 1, reinterpret_cast<uint32_t*>(stage_host + o_sel));
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemcpyAsync(stage_dev, stage_host, total, cudaMemcpyHostToDevice, st) != cudaSuccess) return RLFC_ERR_CUDA;
    uint64_t* dstat = reinterpret_cast<uint64_t*>(stage_dev);
    const int32_t* dslots = reinterpret_cast<const int32_t*>(stage_dev + o_slot);
    const int64_t img = (int64_t)H * W * 3;
    int rc = RLFC_ERR_ARGUMENT;
    // B = 4: one kernel over the prepared record index (k_image_indexed4)
    rlfc_index_view iv;
    if (ws && f->block == 4 && rlfc_staged_index_view(f, ws, ws_bytes, present, &iv) == RLFC_OK)
        rc = rlfc::image_indexed_launch(f, &iv, stop_level, s, t, rgb_dev, (int64_t)W * 3, dstat, stream);
    if (rc == RLFC_ERR_ARGUMENT && ws)
        rc = rlfc::decode_field_staged_sel(f, stop_level, dslots, 0, f->hb, rgb_dev, img, (int64_t)W * 3, ws,
                                           ws_bytes, present, n_flagged,
                                           reinterpret_cast<const int32_t*>(stage_dev + o_rows), 1, dstat, stream,
                                           reinterpret_cast<const uint32_t*>(stage_dev + o_sel), sel_n);
    if (rc == RLFC_ERR_ARGUMENT)
        rc = rlfc_decode_field(f, stop_level, dslots, 0, f->hb, rgb_dev, img, (int64_t)W * 3, dstat, stream);
    if (rc != RLFC_OK) return rc;
    if (cudaMemcpyAsync(rgb_host, rgb_dev, img, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(stage_host, dstat, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return RLFC_ERR_CUDA;
    std::memcpy(status_word, stage_host, 8);
    return RLFC_OK;
}
