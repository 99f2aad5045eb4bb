/*
 * rlfc_b200.h -- C ABI of the B200-native RLFC decode / render hot path.
 *
 * The reference's plugin API for this path is the `rlfc.kernels` module
 * (/root/reference/pkg/src/rlfc/kernels.py), selected at import time
 * (kernels.py:22-44) and called by rlfc.decoder / rlfc.renderer.  Each entry
 * point below replaces one of those calls; the Python host layer
 * (paper_1805_06019_b200/decoder.py, renderer.py) keeps the reference's
 * public signatures and binds these symbols with ctypes.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes; every data pointer is DEVICE memory owned by
 *     the caller (torch tensors in the Python host layer); nothing here
 *     allocates output memory;
 *   - `stream` is a cudaStream_t passed as void*; work is enqueued on it and
 *     the call returns without synchronising;
 *   - the return value is RLFC_OK or RLFC_ERR_ARGUMENT / RLFC_ERR_CUDA for
 *     launch problems.  Stream-format errors are DATA-dependent and are
 *     reported asynchronously through a device status word (below);
 *   - thread-safe: the field descriptor is read-only.
 *
 * Device status word (uint64, caller zero-initialises): 0 = ok.  Otherwise
 *   status = ((RLFC_KEY_MAX - key) << 2) | code
 * where code is 1 (corrupt coded pack) or 2 (descriptor outside range table),
 * mirroring kernels.py:165-171, and key orders failures exactly as the
 * reference encounters them (decoder.py:187-210 image -> channel, then
 * kernels.py:227-237 block row -> block column).  The largest status word is
 * the failure the reference would raise first; decoder._raise_status
 * (decoder.py:66-70) maps the code to its FormatError.
 */
#ifndef RLFC_B200_H
#define RLFC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RLFC_OK 0
#define RLFC_ERR_CORRUPT_PACK 1
#define RLFC_ERR_BAD_DESCRIPTOR 2
#define RLFC_ERR_ARGUMENT 3
#define RLFC_ERR_CUDA 4

#define RLFC_MAX_LEVELS 32
#define RLFC_KEY_MAX (1ull << 60)

/* One parsed stream resident in device memory (decoder.py:20-28
 * DecoderState).  Geometry follows container.py:59-145; the SRV sections
 * are the stream's unmodified bytes (container.py:394-399) copied to HBM
 * with >= 16 zero bytes of tail padding; offsets are the u64 block offset
 * arrays (container.py:382-391); roots are the decoded, unbiased root planes
 * (container.py:355-379), stored (rsx, rsy, 3, hp, wp) as int16 when every
 * sample fits, else int32. */
typedef struct rlfc_field {
    int32_t s_count, t_count, width, height;
    int32_t block, tree_height, quant_shift, m_nodes;
    int32_t wp, hp, wb, hb, rsx, rsy;
    int32_t roots_i16; /* 1: roots are int16, 0: int32 */
    int32_t bitmap_bytes;
    /* Largest compressed size (bytes, all three channels, +32 alignment
     * slack per channel) of any run of TW/block consecutive records inside
     * one block row, TW = 32 pixels (16 for block 16) -- the shared-memory
     * staging need of the fused decode's tiles (host-computed from the
     * offset arrays at init; 0 = unknown). */
    int32_t tile_bytes_max;
    int32_t _reserved;
    /* BFS geometry (container.py:102-145): level l (0..h-1) holds
     * level_sx[l] x level_sy[l] nodes starting at serial index level_base[l]. */
    int32_t level_base[RLFC_MAX_LEVELS];
    int32_t level_sx[RLFC_MAX_LEVELS];
    int32_t level_sy[RLFC_MAX_LEVELS];
    const uint8_t *srv[3];
    const uint64_t *offsets[3];
    uint64_t srv_len[3];
    const void *roots;
} rlfc_field;

/* Random-access block decode, batched.  Replaces kernels.decode_chain_core
 * (kernels.py:162-216) as called by decoder.decode_block_progressive
 * (decoder.py:81-106).  req: n x 6 int32 (s, t, bx, by, channel, stop_level),
 * already range-checked by the host (decoder.py:51-63).  out: n x B*B int32
 * (root block + dequantised chain residuals).  status: n int32 per-request
 * codes (0 / 1 / 2). */
int rlfc_decode_blocks(const rlfc_field *f, const int32_t *req, int32_t n,
                       int32_t *out, int32_t *status, void *stream);

/* One block, synchronously: the random-access latency path of
 * decoder.decode_block / decode_block_progressive (decoder.py:73-112).  The
 * request travels in the kernel parameters; the B*B values followed by the
 * status code (0 / 1 / 2, kernels.py:165-171) land in dev (device, B*B+1
 * int32) and are copied into host (pinned host memory, B*B+1 int32); with
 * dev NULL the kernel writes them straight into host, which must then be
 * pinned and device-addressable (unified addressing).  The call returns after
 * the result is in host: with dev == NULL the kernel writes the block into
 * host, status word last, and the call polls that word (the stream is queried
 * every 1024 polls, so a failed launch returns RLFC_ERR_CUDA instead of
 * hanging); with a device buffer it copies and synchronises the stream.
 * Out-of-range requests return RLFC_ERR_ARGUMENT (the host checks them first,
 * decoder.py:51-63). */
int rlfc_decode_block_sync(const rlfc_field *f, int32_t s, int32_t t,
                           int32_t bx, int32_t by, int32_t channel,
                           int32_t stop_level, int32_t *dev, int32_t *host,
                           void *stream);

/* Single-block requests through a resident server kernel: the latency path
 * of decoder.decode_block / decode_block_progressive (decoder.py:73-112)
 * under a stream of requests.  The mailbox lives in pinned host memory
 * (device-addressable, zero-filled before first use) and belongs to one host
 * thread and one CUDA stream.  rlfc_block_server_request writes the request,
 * launches the server kernel on `stream` when the stream is idle (first
 * request, or the server exited after idle_ns ns without work) and returns
 * once the result is complete in the mailbox, copied to out: out[0 .. B*B)
 * the block, out[B*B] the status (0 / 1 / 2, kernels.py:165-171).  The result
 * arrives as 16-byte chunks {3 values, request number}.  index (nullable) is
 * used by servers launched while it is given.  Out-of-range
 * requests return RLFC_ERR_ARGUMENT.  rlfc_block_server_stop makes a running
 * server exit and waits for it (before the mailbox or the field is
 * released). */
#define RLFC_MAILBOX_STOP 0xFFFFFFFFu
/* Read-only view of a prepared record index (rlfc_staged_index_view): the
 * bitmap words and word slot ranks ([nwp][nrec], word-major), the anomaly
 * flags and the payload entries (payload offset, descriptor) of a workspace
 * prepared by rlfc_staged_prepare.  The block server decodes a B = 4 request
 * of an unflagged record from it (one lane per chain level) instead of
 * walking the record. */
typedef struct rlfc_index_view {
    const uint32_t *bm, *rk, *rec_flag, *entries;
    int64_t nrec;
    int32_t nwp, _pad;
    uint64_t cap;
} rlfc_index_view;
int rlfc_staged_index_view(const rlfc_field *f, void *workspace,
                           uint64_t workspace_bytes, uint64_t present_total,
                           rlfc_index_view *out);
typedef struct rlfc_mailbox {
    uint32_t req_seq;      /* host: request number (written after req) */
    int32_t req[6];        /* s, t, bx, by, channel, stop_level */
    uint32_t req_seq2;     /* host: the request number again, written last */
    uint32_t _pad[8];      /* the host-written words keep their own 64-byte line */
    uint32_t out[88][4];   /* device: result chunks {v[3q], v[3q+1], v[3q+2], request number} */
} rlfc_mailbox;
int rlfc_block_server_request(const rlfc_field *f, rlfc_mailbox *mb,
                              int32_t s, int32_t t, int32_t bx, int32_t by,
                              int32_t channel, int32_t stop_level,
                              uint64_t idle_ns, const rlfc_index_view *index,
                              int32_t *out, void *stream);
int rlfc_block_server_stop(rlfc_mailbox *mb, void *stream);
/* rlfc_block_server_request with its arguments in one caller-owned struct
 * (the host fills req per call): one pointer crosses the FFI boundary. */
typedef struct rlfc_block_call {
    const rlfc_field *f;
    rlfc_mailbox *mb;
    const rlfc_index_view *index;
    void *stream;
    uint64_t idle_ns;
    int32_t *out;
    int32_t req[6]; /* s, t, bx, by, channel, stop_level */
    int32_t _pad[2];
} rlfc_block_call;
int rlfc_block_server_call(const rlfc_block_call *call);

/* Whole padded planes.  Replaces kernels.decode_plane_core
 * (kernels.py:219-242) as called by decoder.decode_plane (decoder.py:165-184).
 * planes: n x 3 int32 (s, t, channel); out: n x hp x wp int32.  Failure key =
 * (request index, block row, block column). */
int rlfc_decode_planes(const rlfc_field *f, int32_t stop_level,
                       const int32_t *planes, int32_t n, int32_t *out,
                       uint64_t *status, void *stream);

/* One padded plane in one call (decoder.decode_plane, decoder.py:165-184):
 * request and status staged through stage_host / stage_dev (pinned / device,
 * 32 bytes each), the plane decoded into plane_dev (hp*wp int32), copied into
 * plane_host (pinned); returns drained, the status word in *status_word.
 * With a prepared record index (rlfc_staged_index_view; B = 4, nullable)
 * every block of an unflagged record is summed from the index
 * (k_plane_indexed4); otherwise, and for flagged records, the record walk of
 * k_decode_planes. */
int rlfc_decode_plane_host(const rlfc_field *f, int32_t stop_level,
                           int32_t s, int32_t t, int32_t channel,
                           int32_t *plane_dev, int32_t *plane_host,
                           uint8_t *stage_host, uint8_t *stage_dev,
                           uint64_t *status_word,
                           const rlfc_index_view *index, void *stream);

/* Fused full-field decode: every (s, t) image with image_slots[s*T + t] >= 0
 * (image_slots NULL = all images, slot = s*T + t), block rows
 * [by_lo, by_hi), all three channels: tree traversal + YCoCg-R inverse +
 * clamp + RGB8 store (decoder.py:187-210 decode_image / decode_all with
 * colorspace.py:27-56).  Output pixel (s, t, y, x) goes to
 *   rgb + slot(s, t) * img_stride + (y - by_lo*B) * row_stride + 3*x
 * for y < height, x < width (the true-dims crop).  Failure key =
 * ((image*3 + channel)*hb + by)*wb + bx with image = s*T + t. */
int rlfc_decode_field(const rlfc_field *f, int32_t stop_level,
                      const int32_t *image_slots, int32_t by_lo, int32_t by_hi,
                      uint8_t *rgb, int64_t img_stride, int64_t row_stride,
                      uint64_t *status, void *stream);

/* Same contract as rlfc_decode_field, computed by the simple per-(image,
 * block) kernel that walks every record once per image exactly like
 * kernels.decode_plane_core.  Kept as the always-applicable path and as the
 * in-library cross-check of the fused kernel. */
int rlfc_decode_field_simple(const rlfc_field *f, int32_t stop_level,
                             const int32_t *image_slots, int32_t by_lo,
                             int32_t by_hi, uint8_t *rgb, int64_t img_stride,
                             int64_t row_stride, uint64_t *status,
                             void *stream);

/* Staged full-field decode: the same contract and output as
 * rlfc_decode_field, computed in two launches per call -- a payload decode
 * (one lane per present payload, kernels.py:128-159 + 202-211) into a
 * residual array, and a blend (residual gather by bitmap rank + YCoCg-R
 * inverse + clamp, colorspace.py:27-56) -- over a record index that
 * rlfc_staged_prepare builds ONCE per workspace: the stream-invariant part
 * of the reference's per-image record walk (kernels.py:162-200: per present
 * node its payload offset and descriptor; per record its slot base, bitmap
 * words and word ranks; anomaly flags), as the reference builds its own
 * init-time index (`chains`, decoder.py:40-44), plus the RGB8 of every root
 * sample.  The workspace (rlfc_decode_workspace_bytes(f, present_total)
 * bytes, 256-byte aligned, caller-owned) also holds the residuals; every
 * call BISE-decodes every present payload of its block-row band.
 * present_total: the number of present nodes over all records
 * (rlfc_count_present).  Returns RLFC_ERR_ARGUMENT when the stream is
 * outside this path's envelope (block 4/8/16, S <= 64, h <= 8, level rows of
 * <= 64 nodes, quantisation shift <= 20, SRV sections < 4 GiB); the caller
 * then uses rlfc_decode_field.  rlfc_staged_prepare (synchronous) also
 * decodes every payload once and lists the records with any stream anomaly
 * (bad descriptor, truncation, corrupt pack); it returns their number in
 * *n_flagged, which each decode call takes back: units touching them are
 * redone by the reference-order walk after the blend, so values and the
 * failure word are identical to rlfc_decode_field's.  t_rows (device,
 * n_trows entries; NULL = every camera row) restricts the blend to the camera
 * rows holding requested views (with an image slot table). */
int rlfc_count_present(const rlfc_field *f, uint64_t *count, void *stream);
int rlfc_decode_workspace_bytes(const rlfc_field *f, uint64_t present_total,
                                uint64_t *bytes);
int rlfc_staged_prepare(const rlfc_field *f, void *workspace,
                        uint64_t workspace_bytes, uint64_t present_total,
                        int32_t *n_flagged, void *stream);
int rlfc_decode_field_staged(const rlfc_field *f, int32_t stop_level,
                             const int32_t *image_slots, int32_t by_lo,
                             int32_t by_hi, uint8_t *rgb, int64_t img_stride,
                             int64_t row_stride, void *workspace,
                             uint64_t workspace_bytes, uint64_t present_total,
                             int32_t n_flagged, const int32_t *t_rows,
                             int32_t n_trows, uint64_t *status,
                             void *stream);

/* Device record directory: the stream-invariant part of the reference's
 * per-image record walk (kernels.py:162-200), done once per stream and GPU
 * (the reference keeps its own init-time index, `chains`, decoder.py:40-44).
 * The present nodes' stream bytes (descriptor + BISE payload, unchanged) are
 * regrouped into tile-major blobs, one per (block row, 64-pixel chunk, tree
 * level, node row):
 *     u32 n | u16 nbits, ntrits | u32 pad[2] | u32 mask[3*nb] | u16 off[n] |
 *     u16 rot[n] | node bytes (pad 16)
 * mask[c*nb + b] = presence bits of the node row in record (c, block b of the
 * chunk) (kernels.py:181-183); off[j] = byte offset of the j-th present node
 * (rank order c, b, x); rot[] = the ranks ordered by BISE mode (plain bits,
 * trits, quints), nbits / ntrits the first two counts.  blob_off[i] is blob i's offset in 16-byte units, blob
 * i = (by * nchunks + chunk) * rows + row_base[l] + tl, with rows = sum of
 * level_sy over the levels (level 0 first).  root_rgb holds the RGB8 of every
 * root sample (colorspace.py:27-56), rows of rgb_stride bytes.  Records with
 * a stream anomaly (descriptor >= 30, a node past the record end,
 * inconsistent offsets) are not in any blob; they are listed in flagged
 * (c * wb*hb + block) and decoded by the reference-order walk.
 *
 * Build: rlfc_dir_plan fills the geometry and the scratch / root_rgb sizes;
 * the caller allocates scratch (scratch_bytes), blob_off (n_blobs + 1 u32),
 * flagged (nrec int32), root_rgb and tables (RLFC_DIR_TABLE_BYTES);
 * rlfc_dir_size (synchronous) sizes the
 * blobs (blob_bytes, n_flagged); the caller allocates blobs (blob_bytes + 64,
 * the tail lets 64-bit bit windows read past the last payload);
 * rlfc_dir_build fills them.  RLFC_ERR_ARGUMENT: outside this path's
 * envelope (block 4, S <= 32, h <= 8, int16 roots, a blob over 64 KiB). */
#define RLFC_DIR_TABLE_BYTES 16384

typedef struct rlfc_dir {
    int32_t tw, nb, nchunks, rows;
    int64_t n_blobs, nrec;
    uint64_t scratch_bytes, root_rgb_bytes;
    int32_t rgb_stride, n_flagged;
    uint64_t blob_bytes;
    void *scratch;
    uint32_t *blob_off;
    int32_t *flagged;
    uint8_t *root_rgb;
    uint8_t *blobs;
    uint8_t *tables;    /* RLFC_DIR_TABLE_BYTES: dequantisation + digit tables */
} rlfc_dir;

int rlfc_dir_plan(const rlfc_field *f, rlfc_dir *d);
int rlfc_dir_size(const rlfc_field *f, rlfc_dir *d, void *stream);
int rlfc_dir_build(const rlfc_field *f, rlfc_dir *d, void *stream);

/* Full-field decode over the record directory (rlfc_dir_build): same
 * contract and output as rlfc_decode_field for all S x T images (no slot
 * table), block rows [by_lo, by_hi).  One persistent kernel per call: TMA
 * prefill of every view's RGB(root) rows, BISE decode of each dirty unit's
 * chain payloads from the blobs (kernels.py:128-159, 202-211), YCoCg-R
 * inverse + clamp (colorspace.py:27-56), TMA store; every payload is
 * decoded in every call.  Records listed as flagged are then re-decoded by
 * the reference-order walk, so values and the failure word equal
 * rlfc_decode_field's.  rgb, img_stride and row_stride must be multiples
 * of 16 bytes. */
int rlfc_decode_field_dir(const rlfc_field *f, const rlfc_dir *d,
                          int32_t stop_level, int32_t by_lo, int32_t by_hi,
                          uint8_t *rgb, int64_t img_stride, int64_t row_stride,
                          uint64_t *status, void *stream);

/* Random-access block decode over a workspace prepared by
 * rlfc_staged_prepare: same requests, outputs and per-request codes as
 * rlfc_decode_blocks (out-of-range requests report 3), but each chain
 * payload is found from its record's bitmap word and word rank and its
 * index entry instead of a walk over the record's earlier nodes
 * (kernels.py:162-216 early-exit walk); anomalous records take the
 * reference-order walk. */
int rlfc_decode_blocks_indexed(const rlfc_field *f, void *workspace,
                               uint64_t workspace_bytes, uint64_t present_total,
                               const int32_t *req, int32_t n, int32_t *out,
                               int32_t *status, void *stream);

/* The reference kernel module's decode entry points with their own
 * arguments (INTEGRATION.md Route 2, paper_1805_06019_b200/kernels_b200.py):
 * rlfc_chain_core is kernels.decode_chain_core (kernels.py:162-216) for n
 * records at once -- SRV bytes (device, srv_len bytes + >= 32 readable pad),
 * record offsets rec_offs[n], the ascending target list (the ancestor
 * chain), out[n][bsq] pre-filled with the root blocks (in/out), status[n]
 * 0 / 1 / 2.  rlfc_plane_core is kernels.decode_plane_core
 * (kernels.py:219-242) for one plane: root_plane / out_plane int32
 * (blocks_y*block, blocks_x*block); *status (caller initialises to
 * UINT64_MAX) becomes (first failing block index << 2) | code, blocks in
 * row-major order, as the reference returns at its first failure. */
int rlfc_chain_core(const uint8_t *srv, uint64_t srv_len,
                    const uint64_t *rec_offs, int32_t n, int32_t m_nodes,
                    int32_t bsq, const int64_t *targets, int32_t nt,
                    int32_t shift, int32_t *out, int32_t *status,
                    void *stream);
/* rlfc_chain_core for ONE request on the latency path (decoder.py:101-104
 * calls decode_chain_core per block): targets (nt <= 16) are read on the
 * host, io is pinned host memory of bsq + 1 int32 -- the root block in, the
 * target residuals out, status (kernels.py:165-171 codes) in io[bsq] written
 * last.  Synchronous: returns after polling that word. */
int rlfc_chain_core_sync(const uint8_t *srv, uint64_t srv_len,
                         uint64_t rec_off, int32_t m_nodes, int32_t bsq,
                         const int64_t *targets, int32_t nt, int32_t shift,
                         int32_t *io, void *stream);
int rlfc_plane_core(const uint8_t *srv, uint64_t srv_len,
                    const uint64_t *offsets, int32_t blocks_x,
                    int32_t blocks_y, int32_t m_nodes, int32_t block,
                    const int64_t *targets, int32_t nt, int32_t shift,
                    const int32_t *root_plane, int32_t *out_plane,
                    uint64_t *status, void *stream);

/* BISE payload decode, batched.  Replaces kernels.bise_decode_core
 * (kernels.py:128-159) / bise.bise_decode (bise.py:108-118).  payload i
 * starts at data + offs[i], has descriptor descs[i] and `count` values;
 * out: n x count uint32; status: n int32 (0 ok / 1 corrupt pack /
 * 2 bad descriptor).  `data` must be readable 8 bytes past every payload. */
int rlfc_bise_decode(const uint8_t *data, const int64_t *offs,
                     const uint8_t *descs, int32_t n, int32_t count,
                     uint32_t *out, int32_t *status, void *stream);

/* Slab-pose rendering (renderer.py:233-276 _render_slab), batched.
 * rgb_field: decoded RGB8 camera images at the stop level, camera (s, t) at
 * rgb_field + slots[s*T + t] * H*W*3 (slots NULL = s*T + t); only the tap
 * cameras of each pose are read.  poses: n x 4 doubles
 * (s, t, has_focal, focal_z); geoms: n plane geometries
 * (lightfield.py:24-43).  out: n x oh x ow x 3 uint8.
 * bg: n x 3 uint8 backgrounds.  IEEE double, reference operation order, no
 * FMA contraction: bit-exact with the reference. */
typedef struct rlfc_render_geom {
    double cam_z, img_z, x0, y0, x1, y1;
} rlfc_render_geom;

int rlfc_render_slab(const uint8_t *rgb_field, const int32_t *slots,
                     int32_t S, int32_t T, int32_t W, int32_t H,
                     const double *poses,
                     const rlfc_render_geom *geoms, const uint8_t *bg,
                     int32_t n, int32_t ow, int32_t oh, uint8_t *out,
                     void *stream);

/* A batch of slab poses in one call (renderer.render_views, renderer.py:
 * 279-305 per pose): tap cameras (floor and ceil of each clamped eye
 * coordinate), slot table and camera rows are built on the host, staged with
 * the HOST arrays poses (n x 4 doubles: s, t, has_focal, focal), geoms and bg
 * in stage_host (pinned, rlfc_render_staging_bytes bytes) and sent to
 * stage_dev (device, same size) with one copy; the staged decode in slot
 * mode (workspace as for rlfc_decode_field_staged, else the fused decode)
 * fills field (device, field_cap images of H*W*3), k_render_slab renders into
 * out (device, n*oh*ow*3), copied into out_host (pinned, nullable); the call
 * returns after the stream has drained,
 * with the decode status word in *status_word (0 = success). */
int rlfc_render_slab_batch(const rlfc_field *f, int32_t stop_level, void *ws,
                           uint64_t ws_bytes, uint64_t present,
                           int32_t n_flagged, const double *poses,
                           const rlfc_render_geom *geoms, const uint8_t *bg,
                           int32_t n, int32_t ow, int32_t oh, uint8_t *field,
                           int32_t field_cap, uint8_t *out,
                           uint8_t *stage_host, uint8_t *stage_dev,
                           uint64_t stage_bytes, uint8_t *out_host,
                           uint64_t *status_word, void *stream);
uint64_t rlfc_render_staging_bytes(const rlfc_field *f, int32_t n);

/* One image in one call (decoder.decode_image, decoder.py:187-194): the
 * slot table and camera row are staged in stage_host (pinned, at least
 * 32 + 4*S*T bytes) and sent to stage_dev with one copy; the staged decode
 * in slot mode (workspace as for rlfc_decode_field_staged, else the fused
 * decode) fills rgb_dev (H*W*3), which is copied into rgb_host (pinned);
 * returns after the stream drained, with the decode status word in
 * *status_word. */
int rlfc_decode_image_host(const rlfc_field *f, int32_t stop_level, void *ws,
                           uint64_t ws_bytes, uint64_t present,
                           int32_t n_flagged, int32_t s, int32_t t,
                           uint8_t *rgb_dev, uint8_t *rgb_host,
                           uint8_t *stage_host, uint8_t *stage_dev,
                           uint64_t stage_bytes, uint64_t *status_word,
                           void *stream);

/* Pinhole-pose rendering (renderer.py:279-305 with ray_to_lf_coords
 * renderer.py:87-116 and sample_quadrilinear renderer.py:147-169).
 * frames: n x 14 doubles (eye[3], look[3], right[3], down[3], half, aspect)
 * as computed by the reference's per-frame numpy code
 * (renderer.py:190-209); rgb_field / slots as for rlfc_render_slab.  status: n int32 (0, or -2 when a ray is parallel
 * to the slab planes -- ValueError in renderer.py:97-98). */
int rlfc_render_pinhole(const uint8_t *rgb_field, const int32_t *slots,
                        int32_t S, int32_t T, int32_t W, int32_t H,
                        const double *frames,
                        const rlfc_render_geom *geoms, const uint8_t *bg,
                        int32_t n, int32_t ow, int32_t oh, uint8_t *out,
                        int32_t *status, void *stream);

/* Camera-need marking for pinhole batches: sets need[s*T + t] = 1 for every
 * tap camera any pixel of the n frames samples (same arithmetic as
 * rlfc_render_pinhole).  need: S*T bytes, caller zero-initialises. */
int rlfc_render_pinhole_needs(int32_t S, int32_t T, int32_t W, int32_t H,
                              const double *frames,
                              const rlfc_render_geom *geoms, int32_t n,
                              int32_t ow, int32_t oh, uint8_t *need,
                              void *stream);

/* Root-view decode at init (container.py:175-195, PNG roots): raw holds
 * nplanes inflated IDAT streams (each height rows of 1 + 2*width filtered
 * bytes, raw_plane bytes apart); rlfc_png_unfilter undoes the PNG scanline
 * filters (None / Sub / Up / Average / Paeth, 2 bytes per pixel) into
 * big-endian 16-bit samples out[plane][height][width] (out_plane apart);
 * *bad becomes 1 on a filter type above 4.  rlfc_root_planes removes the
 * channel bias (0, 256, 256) and scatters plane p (decode order: channel,
 * root row, root column) into the root tensor (rsx, rsy, 3, hp, wp) as int16
 * (i16 = 1) or int32; minmax (nullable, int32[2], caller initialises to
 * {INT_MAX-ish, INT_MIN-ish}) receives the value range. */
int rlfc_png_unfilter(const uint8_t *raw, int64_t raw_plane, int32_t nplanes,
                      int32_t width, int32_t height, uint16_t *out,
                      int64_t out_plane, int32_t *bad, void *stream);
int rlfc_root_planes(const uint16_t *samples, int32_t nplanes, int32_t rsx,
                     int32_t rsy, int32_t hp, int32_t wp, int32_t i16,
                     void *dst, int32_t *minmax, void *stream);

/* Producer side on the GPU (hierarchy.py:182-298 RKV/SRV tree construction,
 * container.py:300-323 records; csrc/rlfc_encode.cu).  rlfc_enc_planes:
 * YCoCg-R of rgb (nimg, h_valid, W, 3) into planes (nimg, 3, hp, wp) int32,
 * zero padded.  rlfc_enc_pyramid: parent (px, py, 3, hp, wp) = floor((sum of
 * weights[cell][m] * member m + 128) / 256) over the <= 4 children of each
 * cell (members x outer, y inner; weights int64 (px*py, 4)).
 * rlfc_enc_srv_level: one tree level top-down -- residual against the
 * reconstructed parent `above`, thresholds, quantise, zigzag, range choice,
 * closed-loop reconstruction written over `planes`; desc [3][nblk][M]
 * (caller fills 0xFF) and zv [3][nblk][M][B*B] receive the coded blocks of
 * the level's nodes (serial index level_base + y*sx + x), *present counts
 * them, *err = 1 when a block exceeds the range table.
 * rlfc_enc_record_sizes / rlfc_enc_records: per record (c*nblk + block)
 * its byte size, then its bytes at rec_off (bitmap, descriptor + BISE
 * payload per present node in BFS order, kernels.py:92-125). */
int rlfc_enc_planes(const uint8_t *rgb, int64_t nimg, int32_t W,
                    int32_t h_valid, int32_t hp, int32_t wp, int32_t *planes,
                    void *stream);
int rlfc_enc_pyramid(const int32_t *child, int32_t sx, int32_t sy,
                     int32_t *parent, int32_t px, int32_t py,
                     const int64_t *weights, int32_t hp, int32_t wp,
                     void *stream);
int rlfc_enc_srv_level(int32_t *planes, const int32_t *above, int32_t sx,
                       int32_t sy, int32_t psy, int32_t hp, int32_t wp,
                       int32_t block, int32_t pixel_threshold,
                       int64_t block_threshold, int32_t shift,
                       int32_t level_base, int32_t m_nodes, uint8_t *desc,
                       uint16_t *zv, uint64_t *present, int32_t *err,
                       void *stream);
int rlfc_enc_record_sizes(const uint8_t *desc, int64_t nrec, int32_t m_nodes,
                          int32_t bsq, uint64_t *size, void *stream);
int rlfc_enc_records(const uint8_t *desc, const uint16_t *zv, int64_t nrec,
                     int32_t m_nodes, int32_t bsq, const uint64_t *rec_off,
                     uint8_t *out, void *stream);

/* Host plumbing for band-pipelined host-buffer decodes (decoder.HostPipeline):
 * an asynchronous strided copy (cudaMemcpy2DAsync), kind 0 host->device,
 * 1 device->host, 2 device->device.  Not part of the reference interface. */
int rlfc_copy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch,
                int64_t width, int64_t height, int32_t kind, void *stream);

/* Library identification: returns the number of kernels this build exposes
 * and writes a short version string. */
int rlfc_version(char *buf, int32_t len);

#ifdef __cplusplus
}
#endif

#endif /* RLFC_B200_H */
