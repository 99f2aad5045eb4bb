/*
 * rlfc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference RLFC decode / render path
 * (/root/reference/pkg/src/rlfc, "rlfc" 0.1.0).  It is the parity checker for
 * the CUDA product path and the CPU baseline timed by bench.py; nothing in the
 * product package links or calls it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs load it.
 *
 * Parity of this restatement is pinned against golden vectors produced by the
 * live reference (tools/make_goldens.py -> tests/golden/), see
 * tests/test_oracle_golden.py.
 *
 * Build: make -C oracle   (gcc -O2 -pthread -ffp-contract=off; no fast-math:
 * the render blend is IEEE double in numpy's exact operation order).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define MODE_BITS 0
#define MODE_TRIT 1
#define MODE_QUINT 2

/* bise.py:22-25 RANGE_CARDINALITIES factored as (mode, low bits);
 * bise.py:28-60 _factor / TABLE_MODE / TABLE_BITS. */
static const uint8_t TABLE_MODE[30] = {0, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0,
                                       2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0};
static const uint8_t TABLE_BITS[30] = {1, 0, 2, 0, 1, 3, 1, 2, 4, 2,  3,  5,  3,  4,  6,
                                       4, 5, 7, 5, 6, 8, 6, 7, 9, 7,  8, 10,  8,  9, 11};

int orc_table_mode(int d) { return (d >= 0 && d < 30) ? TABLE_MODE[d] : -1; }
int orc_table_bits(int d) { return (d >= 0 && d < 30) ? TABLE_BITS[d] : -1; }

/* kernels.py:63-70 payload_bits */
int64_t orc_payload_bits(int mode, int bits, int64_t count) {
    if (mode == MODE_BITS) return count * bits;
    if (mode == MODE_TRIT) return 8 * ((count + 4) / 5) + count * bits;
    return 7 * ((count + 2) / 3) + count * bits;
}

/* kernels.py:83-89 get_bits: bit-serial LSB-first field read */
static inline uint32_t get_bits(const uint8_t *buf, int64_t pos, int nbits) {
    uint32_t v = 0;
    for (int i = 0; i < nbits; ++i) {
        int64_t p = pos + i;
        v |= (uint32_t)((buf[p >> 3] >> (p & 7)) & 1) << i;
    }
    return v;
}

/* kernels.py:128-159 bise_decode_core.  Digits are computed arithmetically;
 * kernels.py:47-60 TRIT_DIGITS / QUINT_DIGITS tabulate exactly
 * (pack / base^i) % base. Returns 0, or 1 on a corrupt pack. */
int orc_bise_decode(const uint8_t *data, int count, int mode, int bits,
                    uint32_t *out) {
    int64_t pos = 0;
    if (mode == MODE_BITS) {
        for (int k = 0; k < count; ++k) {
            out[k] = get_bits(data, pos, bits);
            pos += bits;
        }
        return 0;
    }
    int group = mode == MODE_TRIT ? 5 : 3;
    int pack_bits = mode == MODE_TRIT ? 8 : 7;
    uint32_t pack_max = mode == MODE_TRIT ? 242 : 124;
    uint32_t radix = mode == MODE_TRIT ? 3 : 5;
    for (int g0 = 0; g0 < count; g0 += group) {
        int gn = count - g0 < group ? count - g0 : group;
        uint32_t pack = get_bits(data, pos, pack_bits);
        pos += pack_bits;
        if (pack > pack_max) return 1;
        uint32_t rem = pack;
        for (int i = 0; i < gn; ++i) {
            uint32_t digit = rem % radix;
            rem /= radix;
            uint32_t low = 0;
            if (bits > 0) {
                low = get_bits(data, pos, bits);
                pos += bits;
            }
            out[g0 + i] = (digit << bits) | low;
        }
    }
    return 0;
}

/* kernels.py:162-216 decode_chain_core.  out is pre-filled with the root
 * block; targets ascending BFS indices.  Returns 0 / 1 corrupt pack /
 * 2 descriptor outside range table. */
int orc_decode_chain(const uint8_t *srv, int64_t rec_off, int m_nodes, int bsq,
                     const int64_t *targets, int nt, int shift, int32_t *out) {
    if (nt == 0) return 0;
    uint32_t tmp[256];
    int64_t cursor = rec_off + ((m_nodes + 7) >> 3);
    int64_t last = targets[nt - 1];
    int32_t half = (1 << shift) >> 1;
    int ti = 0;
    for (int node = 0; node < m_nodes; ++node) {
        if (node > last) break;
        int present = (srv[rec_off + (node >> 3)] >> (node & 7)) & 1;
        if (!present) {
            if (ti < nt && targets[ti] == node) {
                ++ti;
                if (ti == nt) return 0;
            }
            continue;
        }
        int desc = srv[cursor];
        if (desc >= 30) return 2;
        int mode = TABLE_MODE[desc], bits = TABLE_BITS[desc];
        int64_t pbytes = (orc_payload_bits(mode, bits, bsq) + 7) >> 3;
        if (ti < nt && targets[ti] == node) {
            int st = orc_bise_decode(srv + cursor + 1, bsq, mode, bits, tmp);
            if (st) return st;
            for (int j = 0; j < bsq; ++j) {
                int32_t z = (int32_t)tmp[j];
                if (z == 0) continue;
                if (z & 1) out[j] -= (((z + 1) >> 1) << shift) + half;
                else out[j] += ((z >> 1) << shift) + half;
            }
            ++ti;
            if (ti == nt) return 0;
        }
        cursor += 1 + pbytes;
    }
    return 0;
}

/* kernels.py:219-242 decode_plane_core */
int orc_decode_plane(const uint8_t *srv, const uint64_t *offsets, int wb,
                     int hb, int m_nodes, int block, const int64_t *targets,
                     int nt, int shift, const int32_t *root_plane,
                     int32_t *out_plane) {
    int bsq = block * block, wp = wb * block;
    int32_t acc[256];
    for (int by = 0; by < hb; ++by)
        for (int bx = 0; bx < wb; ++bx) {
            for (int yy = 0; yy < block; ++yy)
                for (int xx = 0; xx < block; ++xx)
                    acc[yy * block + xx] =
                        root_plane[(int64_t)(by * block + yy) * wp + bx * block + xx];
            int st = orc_decode_chain(srv, (int64_t)offsets[by * wb + bx], m_nodes,
                                      bsq, targets, nt, shift, acc);
            if (st) return st;
            for (int yy = 0; yy < block; ++yy)
                for (int xx = 0; xx < block; ++xx)
                    out_plane[(int64_t)(by * block + yy) * wp + bx * block + xx] =
                        acc[yy * block + xx];
        }
    return 0;
}

/* colorspace.py:27-36 ycocgr_to_rgb + colorspace.py:46-56 clip/uint8 */
static inline uint8_t clamp8(int32_t v) { return v < 0 ? 0 : v > 255 ? 255 : (uint8_t)v; }
static inline void ycocg_px(int32_t y, int32_t co, int32_t cg, uint8_t *rgb) {
    int32_t t = y - (cg >> 1);
    int32_t g = cg + t;
    int32_t b = t - (co >> 1);
    int32_t r = b + co;
    rgb[0] = clamp8(r);
    rgb[1] = clamp8(g);
    rgb[2] = clamp8(b);
}

void orc_ycocgr_to_rgb8(const int32_t *y, const int32_t *co, const int32_t *cg,
                        int64_t n, uint8_t *rgb) {
    for (int64_t i = 0; i < n; ++i) ycocg_px(y[i], co[i], cg[i], rgb + 3 * i);
}

/* A parsed stream (decoder.py:20-28 DecoderState, flattened). */
typedef struct {
    int32_t s_count, t_count, width, height;
    int32_t block, tree_height, quant_shift, m_nodes;
    int32_t wp, hp, wb, hb, rsx, rsy;
    const uint8_t *srv[3];
    const uint64_t *offsets[3];
    const int32_t *roots;   /* (rsx, rsy, 3, hp, wp) unbiased */
    const int64_t *chains;  /* (S, T, h) */
} orc_field;

/* decoder.py:165-184 decode_plane (one image channel, padded dims) */
int orc_field_plane(const orc_field *f, int s, int t, int c, int stop_level,
                    int32_t *out) {
    int h = f->tree_height;
    int64_t plane = (int64_t)f->hp * f->wp;
    const int32_t *root = f->roots +
        ((((int64_t)(s >> h) * f->rsy + (t >> h)) * 3 + c) * plane);
    int nt = h - stop_level;
    if (nt <= 0) {
        memcpy(out, root, plane * sizeof(int32_t));
        return 0;
    }
    const int64_t *targets = f->chains + ((int64_t)s * f->t_count + t) * h;
    return orc_decode_plane(f->srv[c], f->offsets[c], f->wb, f->hb, f->m_nodes,
                            f->block, targets, nt, f->quant_shift, root, out);
}

/* decoder.py:187-194 decode_image: 3 planes, crop, inverse lift, clamp */
int orc_field_image(const orc_field *f, int s, int t, int stop_level,
                    uint8_t *rgb, int32_t *scratch /* 3*hp*wp or NULL */) {
    int64_t plane = (int64_t)f->hp * f->wp;
    int32_t *buf = scratch ? scratch : (int32_t *)malloc(3 * plane * sizeof(int32_t));
    int st = 0;
    for (int c = 0; c < 3 && !st; ++c) st = orc_field_plane(f, s, t, c, stop_level, buf + c * plane);
    if (!st) {
        for (int y = 0; y < f->height; ++y)
            for (int x = 0; x < f->width; ++x) {
                int64_t i = (int64_t)y * f->wp + x;
                ycocg_px(buf[i], buf[plane + i], buf[2 * plane + i],
                         rgb + ((int64_t)y * f->width + x) * 3);
            }
    }
    if (!scratch) free(buf);
    return st;
}

typedef struct {
    const orc_field *f;
    int stop_level, n;
    uint8_t *rgb;
    int *status;
    int next; /* atomic work counter */
} decode_all_job;

static void *decode_all_worker(void *arg) {
    decode_all_job *job = (decode_all_job *)arg;
    const orc_field *f = job->f;
    int64_t img = (int64_t)f->height * f->width * 3;
    int64_t plane = (int64_t)f->hp * f->wp;
    int32_t *scratch = (int32_t *)malloc(3 * plane * sizeof(int32_t));
    for (;;) {
        int i = __atomic_fetch_add(&job->next, 1, __ATOMIC_RELAXED);
        if (i >= job->n) break;
        job->status[i] = orc_field_image(f, i / f->t_count, i % f->t_count,
                                         job->stop_level, job->rgb + i * img, scratch);
    }
    free(scratch);
    return NULL;
}

int orc_nproc(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }

/* decoder.py:197-210 decode_all, parallel over images with nthreads POSIX
 * threads (the reference runs the same per-image work serially; images are
 * independent).  Returns the status of the first failing image in (s, t)
 * order and its flat index in *bad_image. */
int orc_field_decode_all(const orc_field *f, int stop_level, uint8_t *rgb,
                         int nthreads, int64_t *bad_image) {
    int n = f->s_count * f->t_count;
    decode_all_job job = {f, stop_level, n, rgb, (int *)calloc(n, sizeof(int)), 0};
    if (nthreads <= 0) nthreads = orc_nproc();
    if (nthreads > n) nthreads = n;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, decode_all_worker, &job);
    decode_all_worker(&job);
    for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
    int st = 0;
    for (int i = 0; i < n; ++i)
        if (job.status[i]) {
            st = job.status[i];
            if (bad_image) *bad_image = i;
            break;
        }
    free(job.status);
    return st;
}

/* decoder.py:81-106 decode_block_progressive (root block + chain) */
int orc_field_block(const orc_field *f, int s, int t, int bx, int by, int c,
                    int stop_level, int32_t *out) {
    int h = f->tree_height, b = f->block;
    int64_t plane = (int64_t)f->hp * f->wp;
    const int32_t *root = f->roots +
        ((((int64_t)(s >> h) * f->rsy + (t >> h)) * 3 + c) * plane);
    for (int yy = 0; yy < b; ++yy)
        for (int xx = 0; xx < b; ++xx)
            out[yy * b + xx] = root[(int64_t)(by * b + yy) * f->wp + bx * b + xx];
    int nt = h - stop_level;
    if (nt <= 0) return 0;
    const int64_t *targets = f->chains + ((int64_t)s * f->t_count + t) * h;
    return orc_decode_chain(f->srv[c], (int64_t)f->offsets[c][by * f->wb + bx],
                            f->m_nodes, b * b, targets, nt, f->quant_shift, out);
}

/* ---------------------------------------------------------------------------
 * Rendering (renderer.py).  IEEE double, numpy operation order, no FMA
 * (-ffp-contract=off).  Camera images come from the decoded field at the
 * requested stop level (renderer.py:212-218 _camera_rgb: decode_plane x3,
 * inverse lift, clip -- identical values to the uint8 field).
 */
#define SNAP_EPS 1e-9 /* renderer.py:23 */

/* renderer.py:82-84 _snap (Python round() is half-even, like rint) */
static inline double snap(double f) {
    double r = rint(f);
    return fabs(f - r) < SNAP_EPS ? r : f;
}

/* renderer.py:119-131 _axis_taps; returns tap count (zero weights dropped) */
static int axis_taps(double coord, int count, int *idx, double *w) {
    double c = coord < 0.0 ? 0.0 : coord;
    if (c > (double)(count - 1)) c = (double)(count - 1);
    if (count == 1) {
        idx[0] = 0;
        w[0] = 1.0;
        return 1;
    }
    int i0 = (int)floor(c);
    if (i0 > count - 2) i0 = count - 2;
    double f = snap(c - (double)i0);
    int n = 0;
    if (f < 1.0) { idx[n] = i0; w[n] = 1.0 - f; ++n; }
    if (f > 0.0) { idx[n] = i0 + 1; w[n] = f; ++n; }
    return n;
}

/* renderer.py:221-230 _vec_taps (scalar form) */
static inline void vec_tap(double coord, int count, int *i0, double *f) {
    double c = coord < 0.0 ? 0.0 : coord;
    if (c > (double)(count - 1)) c = (double)(count - 1);
    if (count == 1) { *i0 = 0; *f = 0.0; return; }
    double fl = floor(c);
    if (fl > (double)(count - 2)) fl = (double)(count - 2);
    *i0 = (int)fl;
    double fr = c - (double)(*i0);
    double r = rint(fr);
    *f = fabs(fr - r) < SNAP_EPS ? r : fr;
}

/* np.interp(x, arange(n), arange(n)): identity with endpoint clamp
 * (renderer.py:177-178, 246-247; grid_info_for renderer.py:75-79). */
static inline double interp_identity(double x, int n) {
    if (x < 0.0) return 0.0;
    if (x > (double)(n - 1)) return (double)(n - 1);
    return x;
}

typedef struct {
    double cam_z, img_z, x0, y0, x1, y1; /* lightfield.py:24-43 PlaneGeometry */
} orc_geom;

/* renderer.py:233-276 _render_slab for one SlabPose.  field: (S,T,H,W,3)
 * uint8 decoded at the stop level.  Returns 0, or -1 when focal == camera
 * plane (ValueError in renderer.py:175-176). */
int orc_render_slab(const uint8_t *field, int S, int T, int W, int H,
                    const orc_geom *g, double ps, double pt, int ow, int oh,
                    int has_focal, double focal_z, const uint8_t *bg,
                    uint8_t *out) {
    double focal = has_focal ? focal_z : g->img_z;
    if (focal == g->cam_z) return -1;
    double ex = interp_identity(ps, S), ey = interp_identity(pt, T), ez = g->cam_z;
    for (int64_t i = 0; i < (int64_t)ow * oh; ++i) {
        out[3 * i] = bg[0]; out[3 * i + 1] = bg[1]; out[3 * i + 2] = bg[2];
    }
    double s_val = interp_identity(ex, S), t_val = interp_identity(ey, T);
    if (!(0.0 <= ex && ex <= (double)(S - 1) && 0.0 <= ey && ey <= (double)(T - 1)))
        return 0;
    int si[2], ti[2];
    double ws[2], wt[2];
    int ns = axis_taps(snap(s_val), S, si, ws);
    int nt = axis_taps(snap(t_val), T, ti, wt);
    double xw = g->x1 - g->x0, yw = g->y1 - g->y0;
    int64_t img = (int64_t)W * H * 3;
    for (int j = 0; j < oh; ++j) {
        double ty = g->y0 + ((j + 0.5) * yw) / oh;
        for (int i = 0; i < ow; ++i) {
            double tx = g->x0 + ((i + 0.5) * xw) / ow;
            double dx = tx - ex, dy = ty - ey, dz = focal - ez;
            double tp = (g->img_z - ez) / dz;
            double ix = ex + tp * dx, iy = ey + tp * dy;
            if (!(g->x0 <= ix && ix <= g->x1 && g->y0 <= iy && iy <= g->y1)) continue;
            double u = ((ix - g->x0) / xw) * W - 0.5;
            double v = ((iy - g->y0) / yw) * H - 0.5;
            double ru = rint(u), rv = rint(v);
            if (fabs(u - ru) < SNAP_EPS) u = ru;
            if (fabs(v - rv) < SNAP_EPS) v = rv;
            int u0, v0;
            double fu, fv;
            vec_tap(u, W, &u0, &fu);
            vec_tap(v, H, &v0, &fv);
            double acc[3] = {0.0, 0.0, 0.0};
            for (int a = 0; a < ns; ++a)
                for (int b = 0; b < nt; ++b) {
                    const uint8_t *im = field + ((int64_t)si[a] * T + ti[b]) * img;
                    for (int p = 0; p < 2; ++p) {
                        double wu = p ? fu : 1.0 - fu;
                        int gx = u0 + p < W - 1 ? u0 + p : W - 1;
                        for (int q = 0; q < 2; ++q) {
                            double wv = q ? fv : 1.0 - fv;
                            int gy = v0 + q < H - 1 ? v0 + q : H - 1;
                            double w = ((ws[a] * wt[b]) * wu) * wv;
                            const uint8_t *px = im + ((int64_t)gy * W + gx) * 3;
                            for (int c = 0; c < 3; ++c) acc[c] = acc[c] + w * (double)px[c];
                        }
                    }
                }
            uint8_t *o = out + ((int64_t)j * ow + i) * 3;
            for (int c = 0; c < 3; ++c) {
                double fl = floor(acc[c] + 0.5);
                o[c] = fl < 0.0 ? 0 : fl > 255.0 ? 255 : (uint8_t)fl;
            }
        }
    }
    return 0;
}

/* renderer.py:279-305 pinhole branch: per pixel ray_to_lf_coords
 * (renderer.py:87-116) + sample_quadrilinear (renderer.py:147-169).
 * The per-frame basis (renderer.py:190-209: eye, normalised look, right,
 * down, tan(fov/2), aspect) is computed by the caller with numpy, exactly as
 * the reference does.  Returns 0, or -2 when some ray is parallel to the
 * planes (ValueError in renderer.py:97-98). */
int orc_render_pinhole(const uint8_t *field, int S, int T, int W, int H,
                       int B, const orc_geom *g, const double *eye,
                       const double *look, const double *right,
                       const double *down, double half, double aspect, int ow,
                       int oh, const uint8_t *bg, uint8_t *out) {
    int64_t img = (int64_t)W * H * 3;
    (void)B;
    for (int j = 0; j < oh; ++j) {
        double py = ((j + 0.5) / oh) * 2.0 - 1.0;
        for (int i = 0; i < ow; ++i) {
            double px = ((i + 0.5) / ow) * 2.0 - 1.0;
            double d[3];
            for (int c = 0; c < 3; ++c)
                d[c] = (look[c] + ((px * half) * aspect) * right[c]) + (py * half) * down[c];
            uint8_t *o = out + ((int64_t)j * ow + i) * 3;
            o[0] = bg[0]; o[1] = bg[1]; o[2] = bg[2];
            if (fabs(d[2]) < 1e-15) return -2;
            double tc = (g->cam_z - eye[2]) / d[2];
            double cx = eye[0] + tc * d[0], cy = eye[1] + tc * d[1];
            if (!(0.0 <= cx && cx <= (double)(S - 1) && 0.0 <= cy && cy <= (double)(T - 1)))
                continue;
            double s = interp_identity(cx, S), t = interp_identity(cy, T);
            double tt = (g->img_z - eye[2]) / d[2];
            double ix = eye[0] + tt * d[0], iy = eye[1] + tt * d[1];
            if (!(g->x0 <= ix && ix <= g->x1 && g->y0 <= iy && iy <= g->y1)) continue;
            double u = ((ix - g->x0) / (g->x1 - g->x0)) * W - 0.5;
            double v = ((iy - g->y0) / (g->y1 - g->y0)) * H - 0.5;
            s = snap(s); t = snap(t); u = snap(u); v = snap(v);
            int si[2], ti[2], ui[2], vi[2];
            double ws[2], wt[2], wu[2], wv[2];
            int ns = axis_taps(s, S, si, ws), nt = axis_taps(t, T, ti, wt);
            int nu = axis_taps(u, W, ui, wu), nv = axis_taps(v, H, vi, wv);
            double acc[3] = {0.0, 0.0, 0.0};
            for (int a = 0; a < ns; ++a)
                for (int b = 0; b < nt; ++b)
                    for (int p = 0; p < nu; ++p)
                        for (int q = 0; q < nv; ++q) {
                            double w = ((ws[a] * wt[b]) * wu[p]) * wv[q];
                            const uint8_t *pxl = field + ((int64_t)si[a] * T + ti[b]) * img +
                                                 ((int64_t)vi[q] * W + ui[p]) * 3;
                            for (int c = 0; c < 3; ++c) acc[c] = acc[c] + w * (double)pxl[c];
                        }
            for (int c = 0; c < 3; ++c) {
                double fl = floor(acc[c] + 0.5);
                o[c] = fl < 0.0 ? 0 : fl > 255.0 ? 255 : (uint8_t)fl;
            }
        }
    }
    return 0;
}

/* Reference-faithful per-view CPU render cost (renderer.py:233-276 with
 * renderer.py:212-218): decode the <=4 tap cameras' planes for THIS view,
 * then blend.  Used only as the timed CPU baseline. */
int orc_render_slab_decoding(const orc_field *f, const orc_geom *g, double ps,
                             double pt, int ow, int oh, int has_focal,
                             double focal_z, int stop_level, const uint8_t *bg,
                             uint8_t *out, uint8_t *scratch_field /* S*T*H*W*3 */) {
    int S = f->s_count, T = f->t_count;
    double ex = interp_identity(ps, S), ey = interp_identity(pt, T);
    int si[2], ti[2];
    double ws[2], wt[2];
    int ns = axis_taps(snap(ex), S, si, ws), nt = axis_taps(snap(ey), T, ti, wt);
    int64_t img = (int64_t)f->width * f->height * 3;
    for (int a = 0; a < ns; ++a)
        for (int b = 0; b < nt; ++b) {
            int st = orc_field_image(f, si[a], ti[b], stop_level,
                                     scratch_field + ((int64_t)si[a] * T + ti[b]) * img, NULL);
            if (st) return st;
        }
    return orc_render_slab(scratch_field, S, T, f->width, f->height, g, ps, pt, ow, oh,
                           has_focal, focal_z, bg, out);
}
