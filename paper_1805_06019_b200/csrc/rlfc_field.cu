// rlfc_field.cu -- fused, tiled full-field decode (placeholder: routes every
// geometry to the per-block kernel until the tiled kernel lands).
#include "rlfc_field.cuh"

namespace rlfc {
int launch_decode_field_tiled(const rlfc_field&, int, const int32_t*, int, int, uint8_t*, int64_t, int64_t,
                              uint64_t*, cudaStream_t) {
    return RLFC_ERR_ARGUMENT;
}
}  // namespace rlfc
