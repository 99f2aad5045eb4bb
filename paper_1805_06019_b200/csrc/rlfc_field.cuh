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
}  // namespace rlfc
