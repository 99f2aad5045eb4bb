// rlfc_producer.cpp -- native stream producer (synthesis + encoder).
//
// Reproduces, byte for byte, the reference producer of .rlfc streams:
//   lightfield.py:207-302  synthesize_lightfield (integer-hash value noise)
//   hierarchy.py:182-213   build_rkv_tree  (2x2 clusters, /256 fixed point)
//   hierarchy.py:216-298   build_srv_tree  (residual, thresholds, quantiser,
//                                           closed-loop reconstruction)
//   kernels.py:73-125      put_bits / bise_encode_core
//   container.py:269-339   serialize (records, bitmaps, offsets)
// The float64 parts (synthesis coordinates) follow numpy's operation order
// and are compiled with -ffp-contract=off.  Cluster filter weights and
// positions are computed by the Python caller with numpy (producer.py), as
// the reference does, and passed in.  Work is spread over POSIX threads:
// cameras for synthesis, (parent, channel) for the RKV pyramid,
// (node, channel) for residuals and (channel, block row) for records.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

namespace {

int g_threads = 0;

int nthreads() {
    if (g_threads > 0) return g_threads;
    unsigned n = std::thread::hardware_concurrency();
    return n ? (int)n : 1;
}

void parallel_for(int64_t n, const std::function<void(int64_t)>& fn) {
    int nt = (int)std::min<int64_t>(nthreads(), n);
    if (nt <= 1) {
        for (int64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    for (int k = 0; k < nt; ++k)
        pool.emplace_back([&] {
            for (;;) {
                int64_t i = next.fetch_add(1);
                if (i >= n) break;
                fn(i);
            }
        });
    for (auto& th : pool) th.join();
}

// ---- synthesis (lightfield.py:207-302) --------------------------------------

constexpr uint64_t M1 = 0x9E3779B97F4A7C15ull, M2 = 0xC2B2AE3D27D4EB4Full;

inline uint64_t hash64(uint64_t x) {  // lightfield.py:211-215
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

inline int64_t lattice(int64_t ix, int64_t iy, uint64_t salt) {  // :218-220
    uint64_t key = ((uint64_t)ix * M1) ^ ((uint64_t)iy * M2) ^ salt;
    return (int64_t)((hash64(key) >> 24) & 0xFF);
}

// Per-axis precomputation of _value_noise (lightfield.py:223-238): the lattice
// cell and the 16-bit fraction of one coordinate.
struct Axis {
    int64_t i0;
    int64_t f;
};
inline Axis axis_of(double w, double freq) {
    double fw = w * freq;
    double fl = std::floor(fw);
    Axis a;
    a.i0 = (int64_t)fl;
    a.f = (int64_t)std::floor((fw - (double)a.i0) * 65536.0);
    return a;
}

inline int64_t value_noise(const Axis& ax, const Axis& ay, uint64_t salt) {
    int64_t v00 = lattice(ax.i0, ay.i0, salt), v10 = lattice(ax.i0 + 1, ay.i0, salt);
    int64_t v01 = lattice(ax.i0, ay.i0 + 1, salt), v11 = lattice(ax.i0 + 1, ay.i0 + 1, salt);
    int64_t top = v00 * (65536 - ax.f) + v10 * ax.f;
    int64_t bot = v01 * (65536 - ax.f) + v11 * ax.f;
    return (top * (65536 - ay.f) + bot * ay.f) >> 32;
}

}  // namespace

extern "C" {

void prod_set_threads(int n) { g_threads = n; }

// Rows [r0, r1) of every view of the scene; rgb: (S, T, r1-r0, W, 3) uint8.
// The scene is per pixel, so any row band reproduces the full synthesis.
int prod_synthesize_rows(int S, int T, int W, int H, uint64_t seed, int r0, int r1, uint8_t* rgb);

// rgb: (S, T, H, W, 3) uint8
int prod_synthesize(int S, int T, int W, int H, uint64_t seed, uint8_t* rgb) {
    return prod_synthesize_rows(S, T, W, H, seed, 0, H, rgb);
}

int prod_synthesize_rows(int S, int T, int W, int H, uint64_t seed, int r0, int r1, uint8_t* rgb) {
    const int NR = r1 - r0;
    const double x0 = -1.5, y0 = -1.5, x1 = S - 1 + 1.5, y1 = T - 1 + 1.5;
    const double zi = 1.0 - 0.0;
    const double z_bg = zi * 1.12, z_oc = zi * 1.05;
    uint64_t salts[16];
    for (int i = 0; i < 16; ++i) salts[i] = hash64(seed * 0x10001ull + (uint64_t)i);
    std::vector<double> ux(W), uy(H);
    for (int i = 0; i < W; ++i) ux[i] = x0 + ((i + 0.5) * (x1 - x0)) / W;
    for (int j = 0; j < H; ++j) uy[j] = y0 + ((j + 0.5) * (y1 - y0)) / H;
    const double ext = std::max(x1 - x0, y1 - y0);
    const double bg_freq = W / (12.0 * ext), oc_freq = W / (7.0 * ext);
    const double bg_freq3 = bg_freq * 3.0, oc_freq3 = oc_freq * 3.0;
    const double oc_cx = (x0 + x1) / 2.0, oc_cy = (y0 + y1) / 2.0;
    const double oc_hw = 0.17 * (x1 - x0), oc_hh = 0.17 * (y1 - y0);
    const double bg_scale = z_bg / zi, oc_scale = z_oc / zi;
    parallel_for((int64_t)S * T, [&](int64_t st) {
        const int s = (int)(st / T), t = (int)(st % T);
        const double cam_x = (double)s, cam_y = (double)t;
        const double bx_off = (1.0 - bg_scale) * cam_x, by_off = (1.0 - bg_scale) * cam_y;
        const double ox_off = (1.0 - oc_scale) * cam_x, oy_off = (1.0 - oc_scale) * cam_y;
        std::vector<double> wxo(W), wyo(H);
        std::vector<Axis> bxc(W), bxf(W), oxc(W), oxf(W), byc(H), byf(H), oyc(H), oyf(H);
        (void)NR;
        for (int i = 0; i < W; ++i) {
            double wxb = bg_scale * ux[i] + bx_off;
            wxo[i] = oc_scale * ux[i] + ox_off;
            bxc[i] = axis_of(wxb, bg_freq);
            bxf[i] = axis_of(wxb, bg_freq3);
            oxc[i] = axis_of(wxo[i], oc_freq);
            oxf[i] = axis_of(wxo[i], oc_freq3);
        }
        for (int j = r0; j < r1; ++j) {
            double wyb = bg_scale * uy[j] + by_off;
            wyo[j] = oc_scale * uy[j] + oy_off;
            byc[j] = axis_of(wyb, bg_freq);
            byf[j] = axis_of(wyb, bg_freq3);
            oyc[j] = axis_of(wyo[j], oc_freq);
            oyf[j] = axis_of(wyo[j], oc_freq3);
        }
        uint8_t* img = rgb + st * (int64_t)W * NR * 3 - (int64_t)r0 * W * 3;
        for (int j = r0; j < r1; ++j) {
            const bool my = std::fabs(wyo[j] - oc_cy) < oc_hh;
            for (int i = 0; i < W; ++i) {
                const bool inside = my && std::fabs(wxo[i] - oc_cx) < oc_hw;
                for (int c = 0; c < 3; ++c) {
                    uint8_t v;
                    if (inside) {
                        int64_t co = value_noise(oxc[i], oyc[j], salts[6 + 2 * c]);
                        int64_t fi = value_noise(oxf[i], oyf[j], salts[7 + 2 * c]);
                        uint8_t tex = (uint8_t)((co * 3 + fi) / 4);
                        v = (uint8_t)(tex / 2 + (40 + 60 * c));  // uint8 wrap
                    } else {
                        int64_t co = value_noise(bxc[i], byc[j], salts[2 * c]);
                        int64_t fi = value_noise(bxf[i], byf[j], salts[2 * c + 1]);
                        v = (uint8_t)((co * 3 + fi) / 4);
                    }
                    img[((int64_t)j * W + i) * 3 + c] = v;
                }
            }
        }
    });
    return 0;
}

// ---- encoder ----------------------------------------------------------------

static const int CARD[30] = {2,   3,   4,   5,   6,   8,   10,  12,  16,   20,   24,   32,   40,   48,   64,
                             80,  96,  128, 160, 192, 256, 320, 384, 512,  640,  768,  1024, 1280, 1536, 2048};
static const int TMODE[30] = {0, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0,
                              2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0, 2, 1, 0};
static const int TBITS[30] = {1, 0, 2, 0, 1, 3, 1, 2, 4, 2, 3, 5, 3, 4, 6,
                              4, 5, 7, 5, 6, 8, 6, 7, 9, 7, 8, 10, 8, 9, 11};

static int64_t payload_bits(int mode, int bits, int64_t count) {  // kernels.py:63-70
    if (mode == 0) return count * bits;
    if (mode == 1) return 8 * ((count + 4) / 5) + count * bits;
    return 7 * ((count + 2) / 3) + count * bits;
}

static inline int64_t put_bits(uint8_t* buf, int64_t pos, uint32_t value, int nbits) {  // kernels.py:73-80
    for (int i = 0; i < nbits; ++i)
        if ((value >> i) & 1) {
            int64_t p = pos + i;
            buf[p >> 3] |= (uint8_t)(1u << (p & 7));
        }
    return pos + nbits;
}

// kernels.py:92-125 bise_encode_core; out pre-zeroed. Returns bits written.
int64_t prod_bise_encode(const uint32_t* values, int64_t n, int mode, int bits, uint8_t* out) {
    int64_t pos = 0;
    if (mode == 0) {
        for (int64_t k = 0; k < n; ++k) pos = put_bits(out, pos, values[k], bits);
        return pos;
    }
    const int group = mode == 1 ? 5 : 3, radix = mode == 1 ? 3 : 5, pbits = mode == 1 ? 8 : 7;
    const uint32_t mask = (1u << bits) - 1u;
    for (int64_t g0 = 0; g0 < n; g0 += group) {
        int gn = (int)std::min<int64_t>(group, n - g0);
        uint32_t pack = 0, mul = 1;
        for (int i = 0; i < gn; ++i) {
            pack += (values[g0 + i] >> bits) * mul;
            mul *= radix;
        }
        pos = put_bits(out, pos, pack, pbits);
        if (bits > 0)
            for (int i = 0; i < gn; ++i) pos = put_bits(out, pos, values[g0 + i] & mask, bits);
    }
    return pos;
}

struct EncodeResult {
    std::vector<int32_t> roots;          // (rsx, rsy, 3, hp, wp)
    std::vector<uint8_t> srv[3];
    std::vector<uint64_t> offsets[3];
    std::vector<int64_t> present;        // per level
    int error = 0;
};

// Encode a light field.  rgb: (S,T,H,W,3) uint8.  weights: for level
// l = 1..h, parent (cx, cy) (cx outer), 4 slots of member weights in the
// reference member order (x outer, y inner); unused slots are 0.
// Strip form: rgb holds H valid rows; the planes have hp_rows rows (a multiple
// of B, zero beyond H), so a block-aligned row band of a large field can be
// encoded on its own -- every RKV/SRV operation is per pixel or per block
// (hierarchy.py:182-271), and records are per block (container.py:306-323).
void* prod_encode_strip(int S, int T, int W, int H, int hp_rows, const uint8_t* rgb, int h, int B,
                        int pixel_threshold, int64_t block_threshold, int shift, const int64_t* weights);

void* prod_encode(int S, int T, int W, int H, const uint8_t* rgb, int h, int B, int pixel_threshold,
                  int64_t block_threshold, int shift, const int64_t* weights) {
    return prod_encode_strip(S, T, W, H, (H + B - 1) / B * B, rgb, h, B, pixel_threshold, block_threshold, shift,
                             weights);
}

void* prod_encode_strip(int S, int T, int W, int H, int hp_rows, const uint8_t* rgb, int h, int B,
                        int pixel_threshold, int64_t block_threshold, int shift, const int64_t* weights) {
    auto* R = new EncodeResult();
    const int wp = (W + B - 1) / B * B, hp = hp_rows;
    const int wb = wp / B, hb = hp / B, bsq = B * B;
    const int64_t plane = (int64_t)wp * hp;
    auto ldim = [](int n, int l) { return (n + (1 << l) - 1) >> l; };
    // level-0 planes: YCoCg-R of the input, zero padded (hierarchy.py:185-193)
    std::vector<std::vector<int32_t>> lv(h + 1);
    lv[0].assign((int64_t)S * T * 3 * plane, 0);
    parallel_for((int64_t)S * T, [&](int64_t st) {
        const uint8_t* img = rgb + st * (int64_t)W * H * 3;
        int32_t* P = lv[0].data() + st * 3 * plane;
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                const uint8_t* px = img + ((int64_t)y * W + x) * 3;
                int32_t r = px[0], g = px[1], b = px[2];
                int32_t co = r - b, tt = b + (co >> 1), cg = g - tt, yy = tt + (cg >> 1);
                int64_t i = (int64_t)y * wp + x;
                P[i] = yy;
                P[plane + i] = co;
                P[2 * plane + i] = cg;
            }
    });
    // RKV pyramid (hierarchy.py:195-212)
    int64_t woff = 0;
    for (int l = 1; l <= h; ++l) {
        int sx = ldim(S, l - 1), sy = ldim(T, l - 1), px = ldim(S, l), py = ldim(T, l);
        lv[l].assign((int64_t)px * py * 3 * plane, 0);
        const int64_t* wl = weights + woff;
        woff += (int64_t)px * py * 4;
        parallel_for((int64_t)px * py * 3, [&](int64_t job) {
            int c = (int)(job % 3), cell = (int)(job / 3);
            int cx = cell / py, cy = cell % py;
            const int64_t* w = wl + (int64_t)cell * 4;
            const int32_t* members[4];
            int nm = 0;
            for (int x = 2 * cx; x <= 2 * cx + 1; ++x)
                for (int y = 2 * cy; y <= 2 * cy + 1; ++y)
                    if (x < sx && y < sy) members[nm++] = lv[l - 1].data() + (((int64_t)x * sy + y) * 3 + c) * plane;
            int32_t* out = lv[l].data() + (((int64_t)cx * py + cy) * 3 + c) * plane;
            for (int64_t i = 0; i < plane; ++i) {
                int64_t acc = 0;
                for (int m = 0; m < nm; ++m) acc += w[m] * (int64_t)members[m][i];
                out[i] = (int32_t)((acc + 128) >> 8);
            }
        });
    }
    {
        int rsx = ldim(S, h), rsy = ldim(T, h);
        R->roots.assign(lv[h].begin(), lv[h].end());
        (void)rsx;
        (void)rsy;
    }
    // SRV tree, top-down with closed-loop reconstruction (hierarchy.py:274-298).
    // Per (level, node, channel, block): descriptor (0xFF = absent) and the
    // zigzag codes.
    std::vector<int> node_count(h), node_base(h);
    int M = 0;
    for (int l = h - 1; l >= 0; --l) {
        node_base[l] = M;
        node_count[l] = ldim(S, l) * ldim(T, l);
        M += node_count[l];
    }
    const int64_t nblk = (int64_t)wb * hb;
    std::vector<uint8_t> desc((int64_t)M * 3 * nblk, 0xFF);
    std::vector<uint16_t> zv((int64_t)M * 3 * nblk * bsq, 0);
    R->present.assign(h, 0);
    std::vector<int32_t> recon_above = lv[h];
    const int32_t half = shift > 0 ? (1 << (shift - 1)) : 0;
    for (int l = h - 1; l >= 0; --l) {
        int sx = ldim(S, l), sy = ldim(T, l), psy = ldim(T, l + 1);
        std::vector<int32_t> recon((int64_t)sx * sy * 3 * plane);
        std::vector<int64_t> pres((int64_t)sx * sy * 3, 0);
        parallel_for((int64_t)sx * sy * 3, [&](int64_t job) {
            int c = (int)(job % 3), cell = (int)(job / 3);
            int x = cell / sy, y = cell % sy;
            const int32_t* child = lv[l].data() + (((int64_t)x * sy + y) * 3 + c) * plane;
            const int32_t* parent = recon_above.data() + (((int64_t)(x / 2) * psy + y / 2) * 3 + c) * plane;
            int32_t* rec = recon.data() + (((int64_t)x * sy + y) * 3 + c) * plane;
            int node = node_base[l] + y * sx + x;
            uint8_t* dsc = desc.data() + ((int64_t)node * 3 + c) * nblk;
            uint16_t* z = zv.data() + ((int64_t)node * 3 + c) * nblk * bsq;
            int32_t r[256], q[256];
            int64_t npres = 0;
            for (int by = 0; by < hb; ++by)
                for (int bx = 0; bx < wb; ++bx) {
                    int64_t energy = 0;
                    for (int yy = 0; yy < B; ++yy)
                        for (int xx = 0; xx < B; ++xx) {
                            int64_t i = (int64_t)(by * B + yy) * wp + bx * B + xx;
                            int32_t v = child[i] - parent[i];
                            if (std::abs(v) < pixel_threshold) v = 0;
                            r[yy * B + xx] = v;
                            energy += std::abs(v);
                        }
                    const bool present = energy >= block_threshold && energy > 0;
                    int64_t blk = (int64_t)by * wb + bx;
                    uint32_t zmax = 0;
                    for (int k = 0; k < bsq; ++k) {
                        int32_t a = std::abs(r[k]) >> shift;
                        q[k] = r[k] < 0 ? -a : a;
                        if (present) {
                            int64_t zz = q[k] >= 0 ? 2 * (int64_t)q[k] : -2 * (int64_t)q[k] - 1;
                            uint16_t z16 = (uint16_t)(uint32_t)zz;
                            z[blk * bsq + k] = z16;
                            zmax = std::max<uint32_t>(zmax, z16);
                        }
                    }
                    if (present) {
                        int d = 0;
                        while (d < 30 && CARD[d] <= (int)zmax) ++d;
                        if (d == 30) {
                            R->error = 1;  // value outside the range table
                            d = 29;
                        }
                        dsc[blk] = (uint8_t)d;
                        ++npres;
                    }
                    for (int yy = 0; yy < B; ++yy)
                        for (int xx = 0; xx < B; ++xx) {
                            int64_t i = (int64_t)(by * B + yy) * wp + bx * B + xx;
                            int32_t qq = q[yy * B + xx], rh = 0;
                            if (present && qq != 0) {
                                int32_t mag = ((qq < 0 ? -qq : qq) << shift) + half;
                                rh = qq < 0 ? -mag : mag;
                            }
                            rec[i] = parent[i] + rh;
                        }
                }
            pres[job] = npres;
        });
        for (int64_t v : pres) R->present[l] += v;
        recon_above.swap(recon);
    }
    // Records (container.py:300-323): per channel, per block row-major:
    // bitmap + (descriptor, payload) of each present node in BFS order.
    const int nbm = (M + 7) >> 3;
    int pbytes[30];
    for (int d = 0; d < 30; ++d) pbytes[d] = (int)((payload_bits(TMODE[d], TBITS[d], bsq) + 7) >> 3);
    for (int c = 0; c < 3; ++c) {
        std::vector<uint64_t> size(nblk);
        parallel_for(nblk, [&](int64_t blk) {
            uint64_t sz = nbm;
            for (int n = 0; n < M; ++n) {
                uint8_t d = desc[((int64_t)n * 3 + c) * nblk + blk];
                if (d != 0xFF) sz += 1 + pbytes[d];
            }
            size[blk] = sz;
        });
        R->offsets[c].resize(nblk);
        uint64_t pos = 0;
        for (int64_t b = 0; b < nblk; ++b) {
            R->offsets[c][b] = pos;
            pos += size[b];
        }
        R->srv[c].assign(pos, 0);
        parallel_for(nblk, [&](int64_t blk) {
            uint8_t* rec = R->srv[c].data() + R->offsets[c][blk];
            uint8_t* cur = rec + nbm;
            uint32_t vals[256];
            for (int n = 0; n < M; ++n) {
                uint8_t d = desc[((int64_t)n * 3 + c) * nblk + blk];
                if (d == 0xFF) continue;
                rec[n >> 3] |= (uint8_t)(1u << (n & 7));
                *cur++ = d;
                const uint16_t* z = zv.data() + (((int64_t)n * 3 + c) * nblk + blk) * bsq;
                for (int k = 0; k < bsq; ++k) vals[k] = z[k];
                prod_bise_encode(vals, bsq, TMODE[d], TBITS[d], cur);
                cur += pbytes[d];
            }
        });
    }
    return R;
}

int prod_result_error(void* h) { return ((EncodeResult*)h)->error; }
int64_t prod_result_srv_len(void* h, int c) { return (int64_t)((EncodeResult*)h)->srv[c].size(); }
void prod_result_copy(void* h, int c, uint8_t* srv_out, uint64_t* offsets_out) {
    auto* R = (EncodeResult*)h;
    std::memcpy(srv_out, R->srv[c].data(), R->srv[c].size());
    std::memcpy(offsets_out, R->offsets[c].data(), R->offsets[c].size() * 8);
}
void prod_result_roots(void* h, int32_t* out) {
    auto* R = (EncodeResult*)h;
    std::memcpy(out, R->roots.data(), R->roots.size() * 4);
}
void prod_result_present(void* h, int64_t* out) {
    auto* R = (EncodeResult*)h;
    std::memcpy(out, R->present.data(), R->present.size() * 8);
}
void prod_free(void* h) { delete (EncodeResult*)h; }

}  // extern "C"
