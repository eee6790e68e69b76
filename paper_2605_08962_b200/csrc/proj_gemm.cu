// placeholder, replaced below
#include "mux_common.cuh"
extern "C" int mux_proj_scatter(const uint16_t*, const uint16_t*, const uint16_t*, int64_t, int32_t,
                                int32_t, const int64_t*, void* const*, int32_t, void*) {
  mux::set_error("projector not built");
  return MUX_ERR_RUNTIME;
}
