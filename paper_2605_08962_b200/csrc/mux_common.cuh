// Shared helpers for the sm_100a kernels of libmuxb200.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mux_b200.h"

#define MUX_FULL 0xffffffffu

namespace mux {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);

#define MUX_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_status(e_, #call); \
  } while (0)

__host__ __device__ inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

__device__ __forceinline__ int next_pow2(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Exclusive block scan of one int64 per thread (all threads must call).
// `s_warp` is 33 int64 of shared scratch.  Returns the exclusive prefix and
// writes the block total to *total.
__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total, int64_t* s_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(MUX_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t t = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(MUX_FULL, t, o);
      if (lane >= o) t += y;
    }
    s_warp[lane] = t;
  }
  __syncthreads();
  const int64_t base = w ? s_warp[w - 1] : 0;
  *total = s_warp[nw - 1];
  __syncthreads();
  return base + x - v;
}

// Keyed exclusive scan over an array in index order: out[i] = sum of val[j]
// for j < i with key[j] == key[i] (key < 0: skipped, out untouched);
// totals[k] = per-key sum.  K scans of the whole array; K is small (<= 16).
template <typename KeyF, typename ValF, typename OutF>
__device__ void keyed_scan(int n, int K, KeyF key, ValF val, OutF out, int64_t* totals,
                           int64_t* s_warp) {
  for (int k = 0; k < K; ++k) {
    int64_t carry = 0;
    for (int base = 0; base < n; base += blockDim.x) {
      const int i = base + threadIdx.x;
      const bool mine = i < n && key(i) == k;
      const int64_t v = mine ? val(i) : 0;
      int64_t tot;
      const int64_t pre = block_excl_scan(v, &tot, s_warp);
      if (mine) out(i, carry + pre);
      carry += tot;
    }
    if (threadIdx.x == 0) totals[k] = carry;
  }
  __syncthreads();
}

// In-place bitonic sort of s_ord[0..npad) (npad a power of two) by the strict
// order `before(a, b)`; entries >= n must sort last (before() handles them).
template <typename Before>
__device__ void bitonic_sort(int* s_ord, int npad, Before before) {
  for (int k = 2; k <= npad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npad; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int a = s_ord[i], b = s_ord[ixj];
          const bool up = (i & k) == 0;
          if (up ? before(b, a) : before(a, b)) {
            s_ord[i] = b;
            s_ord[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Encoder-group of a modality code (text=0, image=1, video=2, audio=3).
__host__ __device__ __forceinline__ int group_of_mod(int m) {
  return m == 1 || m == 2 ? 0 : (m == 3 ? 1 : -1);
}

// Typed view of the plan blob.
struct Plan {
  int64_t* hdr;
  uint32_t* ticket;  // last-CTA ticket of plan_kernel (zero between launches)
  int32_t *seq, *off, *span, *origin, *origin_pos, *group, *enc, *llm_rank;
  int64_t *arena_off, *enc_off, *stage_off, *llm_row;
  int32_t *bin_fill, *bin_nspan, *bin_of, *chunk_nbins, *chunk_err, *fills, *nspans, *cu;
  int32_t *shard_len, *shard_start;
  int64_t *row_base, *arena_rows, *recv_rows, *stage_rows, *llm_rows;
  int32_t *order, *scratch_a, *scratch_b;
  int64_t *dsrc, *ddst, *drows, *dchunk0;
  int32_t *dgroup, *drank;
  int64_t *rsrc, *rdst, *rrows, *rchunk0;
  int32_t *rgroup, *rrank;
  int64_t *gsrc, *gdst, *grows, *gchunk0;
  int32_t *ggroup, *grank;
  int32_t* lssp_state;
  int64_t* lssp_row;  // [S][MUX_LSSP_MAX]
  int32_t *lp_n, *lp_k, *lp_t0, *lp_len;  // CpHybrid pieces [S][sp]
  int64_t* lp_row;
  int64_t *text_off, *tsrc, *tdst, *trows, *trow0;  // text segments of `me`
};

Plan make_plan(void* base, const mux_plan_layout& L);
// LSSP re-targeting of a step plan (lssp.cu), launched after plan_kernel.
int launch_lssp(const mux_plan_cfg& cfg, const int32_t* lens, const Plan& p, cudaStream_t stream);
int launch_emit(const mux_plan_cfg& cfg, const int32_t* lens, const Plan& p, int G, int eta,
                cudaStream_t stream);
// CpHybrid LLM placement (reshard.cu), then the segment tables (lssp.cu).
int launch_cp_hybrid(const mux_plan_cfg& cfg, const int32_t* lens, const int64_t* ids,
                     const Plan& p, cudaStream_t stream);
Plan make_plan_const(const void* base, const mux_plan_layout& L);

// Upper bounds used by the layout.
inline int max_seq_of(const mux_plan_cfg& c) { return c.n_carry_seqs + (c.S - c.n_carry) + 1; }
inline int lssp_of(const mux_plan_cfg& c) { return c.lssp_sp > 0 ? c.lssp_sp : 0; }
inline int max_ret_of(const mux_plan_cfg& c) { return c.S * (c.sp + 1 + lssp_of(c)) + 1; }
inline int max_disp_of(const mux_plan_cfg& c) { return c.S * (lssp_of(c) > 1 ? lssp_of(c) : 1); }
constexpr int kDefaultChunkBytes = 32768;
// proj_gemm.cu: host-known output bases of a device base array (TMA-store maps).
int out_maps_set(void* const* out_bases_dev, int N, void* const* bases_host, int nb);
// Completion-flag value bit marking a poisoned step (segcopy.cu failure path).
constexpr uint64_t kPoisonBit = 1ull << 63;

}  // namespace mux
