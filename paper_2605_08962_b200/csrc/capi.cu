// C ABI plumbing: thread-local error message and CUDA status mapping.
#include <cstdarg>
#include <cstdio>

#include "mux_common.cuh"

namespace mux {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("CUDA error %s (%s) at %s", cudaGetErrorName(e), cudaGetErrorString(e), where);
  return MUX_ERR_CUDA;
}

}  // namespace mux

extern "C" int mux_version(void) { return 3; }

extern "C" void mux_abi_sizes(int64_t* out) {
  out[0] = (int64_t)sizeof(mux_plan_cfg);
  out[1] = (int64_t)sizeof(mux_plan_layout);
  out[2] = (int64_t)sizeof(mux_proj_group);
}
extern "C" const char* mux_last_error(void) { return mux::g_err; }
