// rlfc_field.cuh -- launcher of the fused, tiled full-field decode kernel.
#pragma once
#include <cuda_runtime.h>
#include "../../include/rlfc_b200.h"

namespace rlfc {
// Returns RLFC_ERR_ARGUMENT when the geometry is outside the tiled kernel's
// envelope (the caller then uses the per-block kernel).
int launch_decode_field_tiled(const rlfc_field& f, int stop_level, const int32_t* slots, int by_lo, int by_hi,
                              uint8_t* rgb, int64_t img_stride, int64_t row_stride, uint64_t* status,
                              cudaStream_t stream);

// The staged decode (rlfc_decode_field_staged) with a slot-mode node list the
// caller built on the host (sel_nodes_host) and copied to sel_dev: sel_n is
// its count (> SEL_MAX: too many, the full payload pass runs). sel_dev null:
// the device builds the list (k_sel_nodes).
int decode_field_staged_sel(const rlfc_field* f, int32_t stop_level, const int32_t* image_slots, int32_t by_lo,
                            int32_t by_hi, uint8_t* rgb, int64_t img_stride, int64_t row_stride, void* workspace,
                            uint64_t workspace_bytes, uint64_t present_total, int32_t n_flagged,
                            const int32_t* t_rows, int32_t n_trows, uint64_t* status, void* stream,
                            const uint32_t* sel_dev, int sel_n);
// Host k_sel_nodes: the distinct chain nodes (levels >= k) of the views,
// ascending, into out[1..]; out[0] and the return value are the count, or
// SEL_NODES_MAX + 1 when there are more. out holds 1 + SEL_NODES_MAX words.
constexpr int SEL_NODES_MAX = 64;
int sel_nodes_host(const rlfc_field& f, int k, const int32_t* views, int nviews, uint32_t* out);
// One camera image (B = 4) from the prepared record index (k_image_indexed4);
// RLFC_ERR_ARGUMENT outside its envelope.
int image_indexed_launch(const rlfc_field* f, const rlfc_index_view* ix, int32_t k, int32_t s, int32_t t,
                         uint8_t* rgb, int64_t row_stride, uint64_t* status, void* stream);
}  // namespace rlfc
