// Projector backward on sm_100a (tcgen05 + TMEM + TMA): the gradient path of the
// adapter fused into the return scatter ("gradient path").
//
// After the gradient return (segcopy which=2) the encoder rank holds G [M, N]:
// dL/dY of its encoder rows in encoder order (N = d_llm).  With X [M, K] the
// projector input (encoder output, K = d_enc) and W [N, K] the nn.Linear weight:
//
//   dX = G . W        [M, K]   proj_scatter_pair_kernel (proj_gemm.cu) with
//                              A = G (K-major over N) and B = W^T, which
//                              wt_transpose_kernel writes into the workspace
//   dW = G^T . X      [N, K]   dw_pair_kernel below: reduction over the M rows,
//                              both operands MN-major straight from G and X
//   db = sum_m G[m,:] [N]      colsum_kernel (fp32 partials over 148 row ranges,
//                              summed in order): one HBM pass over G, on a side
//                              stream beside the two GEMMs.  A sum
//                              warp reading the staged G tiles inside
//                              dw_pair_kernel was measured first: holding each
//                              stage for it halved the GEMM (0.85 vs 0.38 ms)
//
// dw_pair_kernel: CTA pairs (cta_group::2), M256 (rows of dW = N) x N256
// (columns = K) tiles, 64-row K-blocks of G / X by TMA (two 64x64 boxes per
// operand half, 128-byte swizzle, MN-major descriptors).  Work split: the first
// floor(T/P)*P tiles run whole (every pair walks the M rows in the same order,
// so the G and X row blocks are read from HBM once and shared through L2); the
// remaining R tiles are split S = P/R ways over M ("split-K", same-chunk pairs
// adjacent), their fp32 partials summed in a fixed order by dw_reduce_kernel
// (deterministic).  Rows [M, round_up(M, 64)) of G and X are zeroed first
// (pad_rows_kernel): the last K-block must not add stale rows.

#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

#include "mux_common.cuh"
#include "umma.cuh"

namespace mux {
namespace bwd {

constexpr int BK = 64;       // rows of G / X per K-block
constexpr int TN = 256;      // tile rows (dW rows = N) per CTA pair
constexpr int TK = 256;      // tile columns (dW columns = K)
#ifndef MUX_BWD_STAGES
#define MUX_BWD_STAGES 4
#endif
constexpr int STAGES = MUX_BWD_STAGES;
constexpr int HALF_BYTES = 128 * BK * 2;          // one CTA's half of an operand: 16 KB
constexpr int STAGE_BYTES = 2 * HALF_BYTES;       // A half + B half
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);    // 320
constexpr int kStagingBytes = kEpiWarps * 32 * 128;
constexpr int kSmem = STAGES * STAGE_BYTES + 512 + kStagingBytes + 1024;
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;

struct Params {
  CUtensorMap tg;    // G [M_max, N], box 64 x 64
  CUtensorMap tx;    // X [M_max, K], box 64 x 64
  int64_t M_max;
  const int64_t* M_dev;
  int N, K;
  uint16_t* dW;      // [N, K] bf16
  float* part;       // [pairs][TN][TK] fp32 partials of split tiles
  int prefetch;      // L2 prefetch distance in K-blocks (0: off)
  int evict_last;    // L2 policy of the operand loads: 1 evict_last, 0 evict_normal
};

// One unit of a pair's work: tile, K-block range, partial slot (-1: direct).
struct Item {
  int tile, kb0, kb1, slot;
};

struct Split {
  int T, P, W1, R, S, KB;
  __device__ int n_items(int cid) const { return W1 + (R && cid < R * S ? 1 : 0); }
  __device__ Item item(int cid, int w) const {
    if (w < W1) return Item{w * P + cid, 0, KB, -1};
    const int c = cid / R;
    return Item{W1 * P + cid % R, (int)((int64_t)c * KB / S), (int)((int64_t)(c + 1) * KB / S),
                cid};
  }
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void __launch_bounds__(kThreads, 1) dw_pair_kernel(const __grid_constant__ Params P) {
  using namespace umma;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = (int)cluster_id_x(), ncl = (int)n_clusters_x();
  int64_t M = P.M_max;
  if (P.M_dev) {
    const int64_t m = *P.M_dev;
    M = m < M ? (m > 0 ? m : 0) : M;
  }
  const int NK = P.K / TK;
  Split sp;
  sp.T = (P.N / TN) * NK;
  sp.P = ncl;
  sp.W1 = sp.T / ncl;
  sp.R = sp.T - sp.W1 * ncl;
  sp.S = sp.R ? ncl / sp.R : 0;
  sp.KB = (int)((M + BK - 1) / BK);
  const int n_items = sp.n_items(cid);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&P.tg);
    tma_prefetch(&P.tx);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer: this CTA's 128 rows of A (= G columns) and 128
    // columns of B (= X columns) per K-block, each as two 64 x 64 boxes
    // Optional L2 prefetch `prefetch` K-blocks ahead (MUX_BWD_PREFETCH, default
    // off: every prefetch is a second L2 lookup of the same boxes, and the L2,
    // not HBM latency, bounds this kernel — 1358 vs 1140 TFLOP/s without it).
    if (lane == 0) {
      const uint64_t pol = P.evict_last ? policy_evict_last() : policy_evict_normal();
      const int D = P.prefetch;
      int stage = 0;
      uint32_t phase = 0;
      for (int w = 0; w < n_items; ++w) {
        const Item it = sp.item(cid, w);
        const int n0 = (it.tile / NK) * TN + (int)rank * 128;
        const int k0 = (it.tile % NK) * TK + (int)rank * 128;
        for (int kb = it.kb0; kb < it.kb0 + D && kb < it.kb1; ++kb) {
          tma_prefetch_l2_2d(&P.tg, n0, kb * BK);
          tma_prefetch_l2_2d(&P.tg, n0 + 64, kb * BK);
          tma_prefetch_l2_2d(&P.tx, k0, kb * BK);
          tma_prefetch_l2_2d(&P.tx, k0 + 64, kb * BK);
        }
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          if (D && kb + D < it.kb1) {
            const int mp = (kb + D) * BK;
            tma_prefetch_l2_2d(&P.tg, n0, mp);
            tma_prefetch_l2_2d(&P.tg, n0 + 64, mp);
            tma_prefetch_l2_2d(&P.tx, k0, mp);
            tma_prefetch_l2_2d(&P.tx, k0 + 64, mp);
          }
          mbar_wait_bounded(&empty[stage], phase ^ 1, false);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          if (leader) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
          const uint32_t bar = smem_u32(&full[stage]) & kPeerBitMask;
          const int m0 = kb * BK;
          tma_load_2d_pair(sa, &P.tg, bar, n0, m0, pol);
          tma_load_2d_pair(sa + HALF_BYTES / 2, &P.tg, bar, n0 + 64, m0, pol);
          tma_load_2d_pair(sa + HALF_BYTES, &P.tx, bar, k0, m0, pol);
          tma_load_2d_pair(sa + HALF_BYTES + HALF_BYTES / 2, &P.tx, bar, k0 + 64, m0, pol);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (leader): M256 N256 K16, both operands MN-major
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = idesc_bf16_f32_major(2 * 128, TK, 1, 1);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int w = 0; w < n_items; ++w) {
        const Item it = sp.item(cid, w);
        if (it.kb0 == it.kb1) continue;  // empty split: the epilogue writes zeros
        mbar_wait_bounded(&tempty[acc], acc_phase ^ 1, false);
        fence_after();
        const uint32_t d = tmem_base + acc * TK;
        for (int kb = it.kb0; kb < it.kb1; ++kb) {
          mbar_wait_bounded(&full[stage], phase, false);
          fence_after();
          const uint8_t* sa = smem + stage * STAGE_BYTES;
          const uint64_t ad = sdesc_sw128_mn(sa, HALF_BYTES / 2);
          const uint64_t bd = sdesc_sw128_mn(sa + HALF_BYTES, HALF_BYTES / 2);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // 16 rows of G / X = 2048 B per step
            mma_bf16_pair(d, ad + 128 * k, bd + 128 * k, idesc, (kb > it.kb0 || k) ? 1u : 0u);
          mma_commit_pair(&empty[stage], 0x3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair(&tfull[acc], 0x3);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ---- epilogue: TMEM -> bf16 dW rows (whole tiles) or fp32 partials
    const int quarter = warp & 3, colgrp = (warp - 2) >> 2;
    uint4* stg = reinterpret_cast<uint4*>(smem + STAGES * STAGE_BYTES + 512) +
                 (warp - 2) * (32 * 8);
    const uint32_t tempty_leader[2] = {mapa(smem_u32(&tempty[0]), 0),
                                       mapa(smem_u32(&tempty[1]), 0)};
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int w = 0; w < n_items; ++w) {
      const Item it = sp.item(cid, w);
      const int row = (int)rank * 128 + quarter * 32 + lane;  // row of the tile
      const int n = (it.tile / NK) * TN + row;
      const int kc0 = (it.tile % NK) * TK + colgrp * 128;    // first column of this warp
      const bool zero = it.kb0 == it.kb1;
      if (!zero) {
        mbar_wait_bounded(&tfull[acc], acc_phase, false);
        fence_after();
      }
#pragma unroll 1
      for (int sub = 0; sub < 2; ++sub) {
        if (it.slot >= 0) {  // fp32 partial: each lane stores its row's 32 columns
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            uint32_t v[32];
            const int col = colgrp * 128 + sub * 64 + j * 32;
            if (zero) {
#pragma unroll
              for (int c = 0; c < 32; ++c) v[c] = 0u;
            } else {
              tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * TK + col, v);
              tmem_wait_ld();
            }
            uint4* dst = reinterpret_cast<uint4*>(P.part + ((int64_t)it.slot * TN + row) * TK +
                                                  col);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              dst[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t v[32];
          const int col = colgrp * 128 + sub * 64 + j * 32;
          if (zero) {
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = 0u;
          } else {
            tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * TK + col, v);
            tmem_wait_ld();
          }
          uint32_t o[16];
#pragma unroll
          for (int c = 0; c < 16; ++c)
            o[c] = pack_bf16(__uint_as_float(v[2 * c]), __uint_as_float(v[2 * c + 1]));
#pragma unroll
          for (int q = 0; q < 4; ++q)
            stg[lane * 8 + ((j * 4 + q) ^ (lane & 7))] =
                make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
        __syncwarp();
        // four rows per store instruction: lanes 8r'..8r'+7 write row r+r'
        const int c8 = lane & 7;
#pragma unroll 4
        for (int r = 0; r < 32; r += 4) {
          const int rr = r + (lane >> 3);
          const int nn = __shfl_sync(MUX_FULL, n, rr);
          const uint4 val = stg[rr * 8 + (c8 ^ (rr & 7))];
          *reinterpret_cast<uint4*>(P.dW + (int64_t)nn * P.K + kc0 + sub * 64 + c8 * 8) = val;
        }
        __syncwarp();
      }
      if (!zero) {
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync();
  fence_after();
  if (warp == 1) tmem_free_pair<512>(tmem_base);
}

// Split tiles: dW[n, k] = sum over the S partials of its pairs, in chunk order.
__global__ void dw_reduce_kernel(const float* part, int T, int P, int N, int K, uint16_t* dW) {
  const int NK = K / TK;
  const int W1 = T / P, R = T - W1 * P;
  if (!R) return;
  const int S = P / R;
  const int r = blockIdx.x / TN, row = blockIdx.x % TN;
  const int tile = W1 * P + r;
  const int n = (tile / NK) * TN + row;
  const int k0 = (tile % NK) * TK;
  for (int c = threadIdx.x; c < TK; c += blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < S; ++j) s += part[((int64_t)(r + j * R) * TN + row) * TK + c];
    reinterpret_cast<__nv_bfloat16*>(dW)[(int64_t)n * K + k0 + c] = __float2bfloat16_rn(s);
  }
}

// db = column sums of G over its first M rows, deterministic: colsum_kernel
// writes fp32 partials of kColsumSplits row ranges (8 columns per thread,
// 16-byte loads), colsum_reduce_kernel adds them in range order.
constexpr int kColsumSplits = 148;
__global__ void __launch_bounds__(256) colsum_kernel(const uint16_t* G, int64_t M_max,
                                                     const int64_t* M_dev, int N, float* part) {
  int64_t M = M_max;
  if (M_dev) {
    const int64_t m = *M_dev;
    M = m < M ? (m > 0 ? m : 0) : M;
  }
  const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c0 >= N) return;
  const int64_t r0 = M * blockIdx.y / gridDim.y, r1 = M * (blockIdx.y + 1) / gridDim.y;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const uint16_t* p = G + r0 * N + c0;
  int64_t r = r0;
  for (; r + 4 <= r1; r += 4, p += 4 * (int64_t)N) {
    uint4 u[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) u[k] = __ldg(reinterpret_cast<const uint4*>(p + k * (int64_t)N));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t w[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s[2 * j] += __uint_as_float(w[j] << 16);
        s[2 * j + 1] += __uint_as_float(w[j] & 0xffff0000u);
      }
    }
  }
  for (; r < r1; ++r, p += N) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      s[2 * j] += __uint_as_float(w[j] << 16);
      s[2 * j + 1] += __uint_as_float(w[j] & 0xffff0000u);
    }
  }
  float4* o = reinterpret_cast<float4*>(part + (int64_t)blockIdx.y * N + c0);
  o[0] = make_float4(s[0], s[1], s[2], s[3]);
  o[1] = make_float4(s[4], s[5], s[6], s[7]);
}

__global__ void colsum_reduce_kernel(const float* part, int splits, int N, uint16_t* db) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  float s = 0.f;
  for (int j = 0; j < splits; ++j) s += part[(int64_t)j * N + c];
  reinterpret_cast<__nv_bfloat16*>(db)[c] = __float2bfloat16_rn(s);
}

// Zero rows [M, min(round_up(M, 64), M_max)) of a [M_max, width] bf16 buffer.
__global__ void pad_rows_kernel(uint16_t* buf, int64_t M_max, const int64_t* M_dev, int width) {
  int64_t M = M_max;
  if (M_dev) {
    const int64_t m = *M_dev;
    M = m < M ? (m > 0 ? m : 0) : M;
  }
  int64_t end = (M + BK - 1) / BK * BK;
  if (end > M_max) end = M_max;
  const int64_t n = (end - M) * width / 8;  // 16-byte words
  uint4* p = reinterpret_cast<uint4*>(buf + M * width);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(0, 0, 0, 0);
}

__global__ void set_ptr_kernel(void** slot, void* p) { *slot = p; }

// W [N, K] -> Wt [K, N] (64 x 64 tiles through shared memory).
__global__ void wt_transpose_kernel(const uint16_t* W, uint16_t* Wt, int N, int K) {
  __shared__ uint16_t t[64][65];
  const int n0 = blockIdx.y * 64, k0 = blockIdx.x * 64;
  for (int i = threadIdx.y; i < 64; i += blockDim.y)
    t[i][threadIdx.x] = W[(int64_t)(n0 + i) * K + k0 + threadIdx.x];
  __syncthreads();
  for (int i = threadIdx.y; i < 64; i += blockDim.y)
    Wt[(int64_t)(k0 + i) * N + n0 + threadIdx.x] = t[threadIdx.x][i];
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int make_map(CUtensorMap* m, const void* base, int64_t rows, int cols) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return MUX_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, BK};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return MUX_ERR_CUDA;
  }
  return MUX_OK;
}

static int pairs_of(int num_sms) {
  int sms = num_sms;
  if (sms <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms / 2 > 0 ? sms / 2 : 1;
}

struct WsLayout {
  size_t wt, part, bases, colsum, total;
};

static WsLayout ws_layout(int32_t K, int32_t N, int pairs) {

  WsLayout L;
  L.wt = 0;
  size_t o = ((size_t)K * N * 2 + 255) & ~size_t(255);
  L.part = o;
  o += ((size_t)pairs * TN * TK * 4 + 255) & ~size_t(255);
  L.bases = o;  // device pointer table of the dX launch (one entry)
  o += 256;
  L.colsum = o;  // db partials [kColsumSplits][N] fp32
  o += ((size_t)kColsumSplits * N * 4 + 255) & ~size_t(255);
  L.total = o;
  return L;
}

}  // namespace bwd
}  // namespace mux

using namespace mux;

extern "C" size_t mux_proj_backward_workspace(int32_t K, int32_t N, int32_t num_sms) {
  return bwd::ws_layout(K, N, bwd::pairs_of(num_sms)).total;
}

extern "C" int mux_proj_backward(const uint16_t* G, const uint16_t* X, const uint16_t* W,
                                 int64_t M_max, const int64_t* M_dev, int32_t K, int32_t N,
                                 uint16_t* dX, uint16_t* dW, uint16_t* db, void* workspace,
                                 size_t workspace_bytes, int32_t num_sms, void* stream) {
  using namespace bwd;
  if (K <= 0 || N <= 0 || K % TK || N % TN || M_max < 0) {
    set_error("projector backward: need K %% %d == 0 and N %% %d == 0 (K=%d N=%d)", TK, TN, K,
              N);
    return MUX_ERR_VALUE;
  }
  if ((((uintptr_t)G | (uintptr_t)X | (uintptr_t)W | (uintptr_t)workspace) & 15) != 0) {
    set_error("projector backward: operands and workspace must be 16-byte aligned");
    return MUX_ERR_VALUE;
  }
  const int pairs = pairs_of(num_sms);
  const WsLayout L = ws_layout(K, N, pairs);
  if (!workspace || workspace_bytes < L.total) {
    set_error("projector backward: workspace of %zu bytes needed (mux_proj_backward_workspace)",
              L.total);
    return MUX_ERR_VALUE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  uint16_t* Wt = reinterpret_cast<uint16_t*>(ws + L.wt);
  if (M_max == 0) {  // no rows: dW and db are zero
    if (dW) MUX_CUDA(cudaMemsetAsync(dW, 0, (size_t)N * K * 2, s));
    if (db) MUX_CUDA(cudaMemsetAsync(db, 0, (size_t)N * 2, s));
    return MUX_OK;
  }
  // rows past the device count up to the next K-block must read as zero
  pad_rows_kernel<<<64, 256, 0, s>>>(const_cast<uint16_t*>(G), M_max, M_dev, N);
  pad_rows_kernel<<<64, 256, 0, s>>>(const_cast<uint16_t*>(X), M_max, M_dev, K);
  // db runs on a side stream beside the GEMMs (an HBM pass next to two
  // L2/tensor-bound kernels, whose CTAs leave room for it): fork here, join at
  // the end; stream-ordered for the caller and capture-safe (events)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (db) {
    static cudaStream_t s_side[16] = {};
    static cudaEvent_t s_fork[16] = {}, s_join[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 16) dev = 0;
    if (!s_side[dev]) {
      MUX_CUDA(cudaStreamCreateWithFlags(&s_side[dev], cudaStreamNonBlocking));
      MUX_CUDA(cudaEventCreateWithFlags(&s_fork[dev], cudaEventDisableTiming));
      MUX_CUDA(cudaEventCreateWithFlags(&s_join[dev], cudaEventDisableTiming));
    }
    side = s_side[dev];
    ev_fork = s_fork[dev];
    ev_join = s_join[dev];
    MUX_CUDA(cudaEventRecord(ev_fork, s));
    MUX_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    float* part = reinterpret_cast<float*>(ws + L.colsum);
    colsum_kernel<<<dim3((N / 8 + 255) / 256, kColsumSplits), 256, 0, side>>>(G, M_max, M_dev,
                                                                              N, part);
    colsum_reduce_kernel<<<(N + 255) / 256, 256, 0, side>>>(part, kColsumSplits, N, db);
    MUX_CUDA(cudaGetLastError());
    MUX_CUDA(cudaEventRecord(ev_join, side));
  }
  MUX_CUDA(cudaGetLastError());
  if (dX) {  // dX = G . W: the forward pair GEMM with A = G and B = W^T
    wt_transpose_kernel<<<dim3(K / 64, N / 64), dim3(64, 8), 0, s>>>(W, Wt, N, K);
    set_ptr_kernel<<<1, 1, 0, s>>>(reinterpret_cast<void**>(ws + L.bases), dX);
    MUX_CUDA(cudaGetLastError());
    void* host_base[1] = {dX};  // the maps of the TMA-store epilogue must see this dX
    int mst = out_maps_set(reinterpret_cast<void* const*>(ws + L.bases), K, host_base, 1);
    if (mst) return mst;
    mux_proj_group g{G, Wt, nullptr, M_max, M_dev, N, 0, nullptr};
    const int st = mux_proj_scatter_grouped(&g, 1, K, reinterpret_cast<void**>(ws + L.bases),
                                            2 * pairs, stream);
    if (st) return st;
  }
  if (dW) {
    Params P;
    memset(&P, 0, sizeof(P));
    int st = make_map(&P.tg, G, M_max, N);
    if (st) return st;
    st = make_map(&P.tx, X, M_max, K);
    if (st) return st;
    P.M_max = M_max;
    P.M_dev = M_dev;
    P.N = N;
    P.K = K;
    P.dW = dW;
    P.part = reinterpret_cast<float*>(ws + L.part);
    static int pf = -1, el = -1;  // MUX_BWD_PREFETCH / MUX_BWD_EVICT_LAST (tuning)
    if (pf < 0) {
      const char* e = getenv("MUX_BWD_PREFETCH");
      pf = e ? atoi(e) : 0;
      const char* f = getenv("MUX_BWD_EVICT_LAST");
      el = f ? atoi(f) : 0;
    }
    P.prefetch = pf;
    P.evict_last = el;
    static bool attr = false;
    if (!attr) {
      MUX_CUDA(cudaFuncSetAttribute(dw_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSmem));
      attr = true;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(2 * pairs);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = kSmem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    MUX_CUDA(cudaLaunchKernelEx(&lc, dw_pair_kernel, P));
    const int T = (N / TN) * (K / TK);
    if (T % pairs) {
      dw_reduce_kernel<<<(T % pairs) * TN, 256, 0, s>>>(P.part, T, pairs, N, K, dW);
      MUX_CUDA(cudaGetLastError());
    }
  }
  if (db) MUX_CUDA(cudaStreamWaitEvent(s, ev_join, 0));  // join the db side stream
  return MUX_OK;
}
