// Projector GEMM fused with the placeholder scatter (sm_100a, tcgen05 + TMEM + TMA).
//
//   out[rank(m)][row(m), :] = bf16( X[m, :] . W^T + bias )   for m < M
//
// X: encoder output rows in encoder order [M, K]; W: nn.Linear weight [N, K];
// row_dst[m] = (rank << 40) | row names the packed-LLM position of encoder
// row m, on this GPU or on an NVLink peer.  There is no reference kernel: the
// adapter sits between the encoder and the LLM and this
// fuses it with the return scatter.
//
// Two kernels, both persistent and warp-specialised (warp 0 TMA producer,
// warp 1 TMEM owner + single-thread MMA issuer, 8 epilogue warps draining
// two 256-column fp32 TMEM accumulators so the epilogue of tile i overlaps the
// MMAs of tile i+1; tcgen05.ld 32x32b.x32 -> +bias -> bf16 -> row stores):
//   proj_scatter_kernel       one CTA per SM, M128 N256 K16, 4-stage ring of
//                             A 128x64 + B 256x64 (128-byte swizzle)
//   proj_scatter_pair_kernel  (default) CTA pairs, tcgen05.mma.cta_group::2
//                             M256 N256 K16, 5-stage ring of half tiles (below);
//                             a warp's 32 output rows leave by one TMA tensor
//                             store when they are consecutive rows (local or peer)
// Both handle up to two problems (encoder groups) per launch.

#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

#include "mux_common.cuh"
#include "umma.cuh"

namespace mux {
namespace proj {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter, 128 columns each
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kStagingBytes = kEpiWarps * 32 * 128;  // per warp: 32 rows x 128 B
constexpr int kSmem = STAGES * STAGE_BYTES + 256 + kStagingBytes + 1024;
constexpr int64_t kRowMask = (1ll << 40) - 1;

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Up to kMaxGroups independent problems (one per encoder group) share N and
// the output buffers; their tiles are enumerated group after group, so one
// persistent launch covers the whole step.
constexpr int kMaxGroups = 2;
constexpr int kMaxOutMaps = 8;

struct GroupParams {
  CUtensorMap ta[kMaxGroups];  // X_g [M_max_g, K_g]
  CUtensorMap tb[kMaxGroups];  // W_g [N, K_g]
  const uint16_t* bias[kMaxGroups];
  const int64_t* row_dst[kMaxGroups];
  const int64_t* M_dev[kMaxGroups];
  int64_t M_max[kMaxGroups];
  int K[kMaxGroups];
  int n_groups, N;
  void* const* out_bases;
  // completion signal (world > 0): the last CTA publishes epoch+1 to every
  // peer's flag slot `me`, as mux_signal does, after every CTA's stores
  uint64_t* const* flags_peers;
  uint64_t* epoch_ctr;
  uint32_t* ticket;  // zero before the first launch; re-armed by the last CTA
  int me, world;
  // optional "consumed" signal at kernel start (E channel, relaxed stores; the
  // kernels before this one in the stream only read the receive windows)
  uint64_t* const* e_flags_peers;
  uint64_t* e_epoch_ctr;
  // status word of the path (nullable): nonzero = poisoned step (segcopy.cu):
  // compute nothing, publish the epoch with kPoisonBit
  const int32_t* poison;
  // TMA-store epilogue (pair kernel, MUX_EPI_TMA): one tensor map per output
  // base, local or NVLink peer (box 64 x 32 rows, 128-byte swizzle = the staging
  // layout); a warp's 32 rows go out in one store when they are consecutive rows
  // of one base (a sample's rows are contiguous in its packed sequence, so nearly
  // all are), else row by row as before
  int epi_tma, n_out;
  CUtensorMap tout[kMaxOutMaps];
  const void* tout_base[kMaxOutMaps];  // the base each map was built for
};

__device__ __forceinline__ bool is_poisoned(const GroupParams& P) {
  return P.poison && *(volatile const int32_t*)P.poison != 0;
}

// E signal by one thread at kernel start (see GroupParams).
__device__ __forceinline__ void consumed_signal(const GroupParams& P) {
  if (!P.e_flags_peers) return;
  const uint64_t e = *P.e_epoch_ctr + 1;
  *P.e_epoch_ctr = e;
  for (int r = 0; r < P.world; ++r) {
    uint64_t* f = P.e_flags_peers[r] + P.me;
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
  }
}

struct TileMap {
  int64_t tiles[kMaxGroups + 1];  // first tile of each group, then the total
  int64_t M[kMaxGroups];
  int kblocks[kMaxGroups];
  int num_m[kMaxGroups], stride[kMaxGroups];
};

__device__ __forceinline__ int gcd_int(int a, int b) {
  while (b) {
    const int t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Row blocks are visited in a golden-ratio stride order (a permutation of
// 0..num_m-1).  Encoder rows are in origin-rank order, so the rows bound for
// one NVLink peer form contiguous blocks; visiting them in order would leave
// all remote stores to one stretch (the tail, on rank 0) with nothing to hide
// behind.  Spread out, they overlap the MMAs of local blocks.  The N-tiles of
// a row block stay adjacent, so the A tile is still shared through L2.
__device__ __forceinline__ int block_stride(int num_m) {
  if (num_m <= 2) return 1;
  int s = (int)(num_m * 0.6180339887) | 1;
  while (gcd_int(s, num_m) != 1) s += 2;
  return s % num_m;
}

__device__ __forceinline__ void locate(const TileMap& tm, int n_groups, int num_n, int64_t tile,
                                       int& g, int& m_blk, int& n_blk) {
  g = 0;
  while (g + 1 < n_groups && tile >= tm.tiles[g + 1]) ++g;
  const int64_t t = tile - tm.tiles[g];
  m_blk = (int)(((t / num_n) * tm.stride[g]) % tm.num_m[g]);
  n_blk = (int)(t % num_n);
}

__global__ void __launch_bounds__(kThreads, 1)
    proj_scatter_kernel(const __grid_constant__ GroupParams P) {
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
  const int N = P.N, num_n = N / BN, G = P.n_groups;
  TileMap tm;
  tm.tiles[0] = 0;
  for (int g = 0; g < G; ++g) {
    int64_t M = P.M_max[g];
    if (P.M_dev[g]) {
      const int64_t m = *P.M_dev[g];
      M = m < M ? (m > 0 ? m : 0) : M;
    }
    tm.M[g] = M;
    tm.kblocks[g] = P.K[g] / BK;
    tm.num_m[g] = (int)((M + BM - 1) / BM);
    tm.stride[g] = block_stride(tm.num_m[g]);
    tm.tiles[g + 1] = tm.tiles[g] + (int64_t)tm.num_m[g] * num_n;
  }
  const bool poisoned = is_poisoned(P);
  const int64_t num_tiles = poisoned ? 0 : tm.tiles[G];

  if (warp == 0 && lane == 0) {
    if (blockIdx.x == 0) consumed_signal(P);
    for (int g = 0; g < G; ++g) {
      tma_prefetch(&P.ta[g]);
      tma_prefetch(&P.tb[g]);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32 * kEpiWarps);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // A (128-row block) is re-read by the 16 N-tiles that run concurrently on other
      // CTAs and W (10.5 MB) by every tile: keep both in L2.
      const uint64_t pol_a = policy_evict_last(), pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int g, m_blk, n_blk;
        locate(tm, G, num_n, tile, g, m_blk, n_blk);
        const CUtensorMap* ta = &P.ta[g];
        const CUtensorMap* tb = &P.tb[g];
        for (int kb = 0; kb < tm.kblocks[g]; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sa, ta, &full[stage], kb * BK, m_blk * BM, pol_a);
          tma_load_2d(sa + A_BYTES, tb, &full[stage], kb * BK, n_blk * BN, pol_b);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int g, m_blk, n_blk;
        locate(tm, G, num_n, tile, g, m_blk, n_blk);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < tm.kblocks[g]; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint8_t* sa = smem + stage * STAGE_BYTES;
          const uint64_t ad = sdesc_sw128(sa), bd = sdesc_sw128(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // +32 B per K16 step inside the swizzle atom
            mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // Epilogue, 8 warps: warp w drains TMEM lane quarter w%4 and one half of
    // the tile's 256 columns, 64 columns per round: TMEM -> registers (+bias,
    // bf16) -> warp-private smem staging (XOR-swizzled, conflict-free) ->
    // coalesced 128-byte row segments (4 rows per store instruction) to each
    // row's destination, local or NVLink peer.  Twice the storing warps of a
    // 4-warp epilogue keeps more peer writes in flight.
    const int quarter = warp & 3, colgrp = (warp - 2) >> 2;
    uint4* stage = reinterpret_cast<uint4*>(smem + STAGES * STAGE_BYTES + 256) +
                   (warp - 2) * (32 * 8);  // [32 rows][8 x uint4] = 4 KB per warp
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int g, m_blk, n_blk;
      locate(tm, G, num_n, tile, g, m_blk, n_blk);
      const uint16_t* bias = P.bias[g];
      const int64_t m = (int64_t)m_blk * BM + quarter * 32 + lane;
      char* my_dst = nullptr;
      if (m < tm.M[g]) {
        const int64_t rd = P.row_dst[g] ? P.row_dst[g][m] : m;  // NULL: row m of base 0
        my_dst = static_cast<char*>(P.out_bases[rd >> 40]) +
                 ((rd & kRowMask) * N + (int64_t)n_blk * BN + colgrp * 128) * 2;
      }
      mbar_wait(&tfull[acc], acc_phase);
      fence_after();
#pragma unroll 1
      for (int sub = 0; sub < 2; ++sub) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t v[32];
          const int col = colgrp * 128 + sub * 64 + j * 32;
          tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + col, v);
          tmem_wait_ld();
          const int n0 = n_blk * BN + col;
          uint32_t o[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            float x0 = __uint_as_float(v[2 * c]), x1 = __uint_as_float(v[2 * c + 1]);
            if (bias) {
              const uint32_t bb = __ldg(reinterpret_cast<const uint32_t*>(bias + n0 + 2 * c));
              x0 += __uint_as_float(bb << 16);
              x1 += __uint_as_float(bb & 0xffff0000u);
            }
            o[c] = pack_bf16(x0, x1);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            stage[lane * 8 + ((j * 4 + q) ^ (lane & 7))] =
                make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
        __syncwarp();
        // four rows per store instruction: lanes 8r'..8r'+7 write row r+r'
        const int c8 = lane & 7;
#pragma unroll 4
        for (int r = 0; r < 32; r += 4) {
          const int row = r + (lane >> 3);
          char* d = reinterpret_cast<char*>(__shfl_sync(MUX_FULL, (unsigned long long)my_dst, row));
          const uint4 val = stage[row * 8 + (c8 ^ (row & 7))];
          if (d) *reinterpret_cast<uint4*>(d + sub * 128 + c8 * 16) = val;
        }
        __syncwarp();
      }
      fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  fence_before();
  if (P.world > 0) __threadfence_system();  // this thread's (peer) row stores first
  __syncthreads();
  fence_after();
  if (warp == 1) tmem_free<512>(tmem_base);
  if (P.world > 0 && warp == 0) {
    __shared__ bool s_last;
    if (lane == 0) s_last = atomicAdd(P.ticket, 1u) == gridDim.x - 1;
    __syncwarp();
    if (s_last) {
      const uint64_t e = *P.epoch_ctr + 1;
      __syncwarp();
      if (lane == 0) {
        *P.ticket = 0;
        *P.epoch_ctr = e;
      }
      __threadfence_system();
      const uint64_t v = poisoned ? (e | kPoisonBit) : e;
      if (lane < P.world) {
        uint64_t* f = P.flags_peers[lane] + P.me;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
      }
    }
  }
}

// ---- CTA-pair variant (cta_group::2; the default, MUX_GEMM_2CTA=0 selects the
// single-CTA kernel above) ------------------------------------------------------
// A cluster of two CTAs on one TPC computes 256 x 256 output tiles with
// tcgen05.mma.cta_group::2 (M256 N256 K16) issued by the leader: each CTA
// stages its 128-row half of A and its 128-column half of B, so a stage is
// 32 KB instead of 48 KB (ring depth MUX_PAIR_STAGES, default 5); both CTAs' TMA loads
// complete on the leader's full barrier; the MMA commits multicast to both
// CTAs' empty/tfull barriers; each CTA drains its own 128 TMEM lanes and
// arrives on the leader's tempty barrier.
#ifndef MUX_PAIR_STAGES
#define MUX_PAIR_STAGES 5  // 5 vs 6: +0.8-0.9% at 1 and 4 GPUs; 4 is slower
#endif
constexpr int BM2 = 256, STAGES2 = MUX_PAIR_STAGES;
constexpr int A2_BYTES = 128 * BK * 2;
constexpr int B2_BYTES = 128 * BK * 2;
constexpr int STAGE2_BYTES = A2_BYTES + B2_BYTES;
#ifndef MUX_EPI_TMA
#define MUX_EPI_TMA 1
#endif
constexpr int kStage2Off = MUX_EPI_TMA ? 1024 : 256;  // staging after the barriers (1 KB-aligned for TMA)
// epilogue staging buffers per warp: 2 lets a sub-block's TMA store still read
// one buffer while the next sub-block fills the other (needs a 5-stage ring)
#ifndef MUX_EPI_BUFS
#define MUX_EPI_BUFS 1
#endif
constexpr int kEpiBufs = MUX_EPI_BUFS;
constexpr int kSmem2 = STAGES2 * STAGE2_BYTES + kStage2Off + kEpiBufs * kStagingBytes + 1024;
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;

__global__ void __launch_bounds__(kThreads, 1)
    proj_scatter_pair_kernel(const __grid_constant__ GroupParams P) {
  using namespace umma;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* tfull = empty + STAGES2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t cid = cluster_id_x(), ncl = n_clusters_x();
  const int N = P.N, num_n = N / BN, G = P.n_groups;
  TileMap tm;
  tm.tiles[0] = 0;
  for (int g = 0; g < G; ++g) {
    int64_t M = P.M_max[g];
    if (P.M_dev[g]) {
      const int64_t m = *P.M_dev[g];
      M = m < M ? (m > 0 ? m : 0) : M;
    }
    tm.M[g] = M;
    tm.kblocks[g] = P.K[g] / BK;
    tm.num_m[g] = (int)((M + BM2 - 1) / BM2);
    tm.stride[g] = block_stride(tm.num_m[g]);
    tm.tiles[g + 1] = tm.tiles[g] + (int64_t)tm.num_m[g] * num_n;
  }
  // the poison decision must be the same in both CTAs of a pair (the leader's
  // MMAs wait for the peer's loads): the leader reads it, the peer copies it
  __shared__ uint32_t s_poison;
  if (threadIdx.x == 0 && leader) s_poison = is_poisoned(P) ? 1u : 0u;

  if (warp == 0 && lane == 0) {
    if (blockIdx.x == 0) consumed_signal(P);
    for (int g = 0; g < G; ++g) {
      tma_prefetch(&P.ta[g]);
      tma_prefetch(&P.tb[g]);
    }
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);  // one arrival per epilogue warp of each CTA
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const bool poisoned = ld_shared_cluster_u32(mapa(smem_u32(&s_poison), 0)) != 0;
  const int64_t num_tiles = poisoned ? 0 : tm.tiles[G];

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = cid; tile < num_tiles; tile += ncl) {
        int g, m_blk, n_blk;
        locate(tm, G, num_n, tile, g, m_blk, n_blk);
        for (int kb = 0; kb < tm.kblocks[g]; ++kb) {
          mbar_wait_bounded(&empty[stage], phase ^ 1, false);
          uint8_t* sa = smem + stage * STAGE2_BYTES;
          if (leader) mbar_expect_tx(&full[stage], 2 * STAGE2_BYTES);
          const uint32_t bar = smem_u32(&full[stage]) & kPeerBitMask;
          tma_load_2d_pair(sa, &P.ta[g], bar, kb * BK, m_blk * BM2 + (int)rank * 128, pol);
          tma_load_2d_pair(sa + A2_BYTES, &P.tb[g], bar, kb * BK, n_blk * BN + (int)rank * 128,
                           pol);
          if (++stage == STAGES2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = idesc_bf16_f32(BM2, BN);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int64_t tile = cid; tile < num_tiles; tile += ncl) {
        int g, m_blk, n_blk;
        locate(tm, G, num_n, tile, g, m_blk, n_blk);
        mbar_wait_bounded(&tempty[acc], acc_phase ^ 1, false);
        fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < tm.kblocks[g]; ++kb) {
          mbar_wait_bounded(&full[stage], phase, false);
          fence_after();
          const uint8_t* sa = smem + stage * STAGE2_BYTES;
          const uint64_t ad = sdesc_sw128(sa), bd = sdesc_sw128(sa + A2_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_pair(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          mma_commit_pair(&empty[stage], 0x3);
          if (++stage == STAGES2) {
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
    const int quarter = warp & 3, colgrp = (warp - 2) >> 2;
    uint4* stage_w = reinterpret_cast<uint4*>(smem + STAGES2 * STAGE2_BYTES + kStage2Off) +
                     (warp - 2) * (32 * 8 * kEpiBufs);
    const uint32_t tempty_leader[2] = {mapa(smem_u32(&tempty[0]), 0),
                                       mapa(smem_u32(&tempty[1]), 0)};
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t tile = cid; tile < num_tiles; tile += ncl) {
      int g, m_blk, n_blk;
      locate(tm, G, num_n, tile, g, m_blk, n_blk);
      const uint16_t* bias = P.bias[g];
      const int64_t m = (int64_t)m_blk * BM2 + (int)rank * 128 + quarter * 32 + lane;
      char* my_dst = nullptr;
      int64_t my_rd = -1;
      if (m < tm.M[g]) {
        const int64_t rd = P.row_dst[g] ? P.row_dst[g][m] : m;  // NULL: row m of base 0
        my_rd = rd;
        my_dst = static_cast<char*>(P.out_bases[rd >> 40]) +
                 ((rd & kRowMask) * N + (int64_t)n_blk * BN + colgrp * 128) * 2;
      }
#if MUX_EPI_TMA
      // the warp's 32 rows are consecutive rows of one output base: one TMA store
      const int64_t rd0 = __shfl_sync(MUX_FULL, my_rd, 0);
      const bool tma_ok = P.epi_tma && (rd0 >> 40) < P.n_out &&
                          __all_sync(MUX_FULL, my_rd >= 0 && my_rd == rd0 + lane) &&
                          P.out_bases[rd0 >> 40] == P.tout_base[rd0 >> 40];
#endif
      mbar_wait_bounded(&tfull[acc], acc_phase, false);
      fence_after();
#pragma unroll 1
      for (int sub = 0; sub < 2; ++sub) {
        uint4* stage = stage_w + (kEpiBufs == 2 ? sub * (32 * 8) : 0);
#if MUX_EPI_TMA
        // the TMA store that last used this buffer has read it
        if (lane == 0) bulk_wait_read_n<kEpiBufs - 1>();
        __syncwarp();
#endif
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t v[32];
          const int col = colgrp * 128 + sub * 64 + j * 32;
          tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + col, v);
          tmem_wait_ld();
          const int n0 = n_blk * BN + col;
          uint32_t o[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            float x0 = __uint_as_float(v[2 * c]), x1 = __uint_as_float(v[2 * c + 1]);
            if (bias) {
              const uint32_t bb = __ldg(reinterpret_cast<const uint32_t*>(bias + n0 + 2 * c));
              x0 += __uint_as_float(bb << 16);
              x1 += __uint_as_float(bb & 0xffff0000u);
            }
            o[c] = pack_bf16(x0, x1);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            stage[lane * 8 + ((j * 4 + q) ^ (lane & 7))] =
                make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
#if MUX_EPI_TMA
        if (tma_ok) {
          fence_proxy_async_smem();  // the staging writes, visible to the TMA engine
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&P.tout[rd0 >> 40], smem_u32(stage),
                         n_blk * BN + colgrp * 128 + sub * 64, (int)(rd0 & kRowMask));
            bulk_commit();
          }
          continue;
        }
#endif
        __syncwarp();
        const int c8 = lane & 7;
#pragma unroll 4
        for (int r = 0; r < 32; r += 4) {
          const int row = r + (lane >> 3);
          char* dd = reinterpret_cast<char*>(__shfl_sync(MUX_FULL, (unsigned long long)my_dst, row));
          const uint4 val = stage[row * 8 + (c8 ^ (row & 7))];
          if (dd) *reinterpret_cast<uint4*>(dd + sub * 128 + c8 * 16) = val;
        }
        __syncwarp();
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
#if MUX_EPI_TMA
  if (warp >= 2 && lane == 0) {
    bulk_wait_all();  // every TMA store of this warp has completed
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
#endif
  fence_before();
  if (P.world > 0) __threadfence_system();
  __syncthreads();
  cluster_sync();  // the peer's MMAs (issued by the leader) are done with this TMEM
  fence_after();
  if (warp == 1) tmem_free_pair<512>(tmem_base);
  if (P.world > 0 && warp == 0) {
    __shared__ bool s_last;
    if (lane == 0) s_last = atomicAdd(P.ticket, 1u) == gridDim.x - 1;
    __syncwarp();
    if (s_last) {
      const uint64_t e = *P.epoch_ctr + 1;
      __syncwarp();
      if (lane == 0) {
        *P.ticket = 0;
        *P.epoch_ctr = e;
      }
      __threadfence_system();
      const uint64_t v = poisoned ? (e | kPoisonBit) : e;
      if (lane < P.world) {
        uint64_t* f = P.flags_peers[lane] + P.me;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
      }
    }
  }
}

// --- host: tensor maps through the driver entry point (no -lcuda link) --------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static int make_map_box(CUtensorMap* m, const void* base, int64_t rows, int cols, int box_cols,
                        int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return MUX_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (output) failed (%d)", (int)r);
    return MUX_ERR_CUDA;
  }
  return MUX_OK;
}

// Output tensor maps of the TMA-store epilogue, cached per device base array
// (out_bases) and N.  The kernel uses a map only while out_bases[r] still equals
// the base the map was built for (tout_base), so a stale entry falls back to the
// row stores instead of writing elsewhere; out_maps_set refreshes an entry from
// host-known bases (the projector backward's per-call dX).
struct OutMaps {
  const void* key;
  int N, n;
  const void* base[kMaxOutMaps];
  CUtensorMap m[kMaxOutMaps];
};
static OutMaps g_out_maps[16];
static int g_n_out_maps = 0;

static int out_maps_build(OutMaps& o, const void* key, int N, void* const* bases, int nb) {
  o.key = key;
  o.N = N;
  o.n = nb;
  for (int r = 0; r < nb; ++r) {
    o.base[r] = bases[r];
    int st = make_map_box(&o.m[r], bases[r], 1ll << 30, N, 64, 32);
    if (st) return st;
  }
  return MUX_OK;
}

static OutMaps* out_maps_find(const void* key, int N) {
  for (int c = 0; c < g_n_out_maps; ++c)
    if (g_out_maps[c].key == key && g_out_maps[c].N == N) return &g_out_maps[c];
  return nullptr;
}

static OutMaps* out_maps_slot(const void* key, int N) {
  OutMaps* o = out_maps_find(key, N);
  if (o) return o;
  return &g_out_maps[g_n_out_maps < 16 ? g_n_out_maps++ : 15];
}

// lookup, reading the base pointers back once for a new array
static int out_maps_lookup(void* const* out_bases, int N, int nb, const OutMaps** out) {
  OutMaps* o = out_maps_find(out_bases, N);
  if (!o || o->n != nb) {
    void* hb[kMaxOutMaps];
    MUX_CUDA(cudaMemcpy(hb, out_bases, nb * sizeof(void*), cudaMemcpyDeviceToHost));
    o = out_maps_slot(out_bases, N);
    int st = out_maps_build(*o, out_bases, N, hb, nb);
    if (st) return st;
  }
  *out = o;
  return MUX_OK;
}

}  // namespace proj

// host-known bases for a device base array (proj_bwd.cu: dX of this call)
int out_maps_set(void* const* out_bases_dev, int N, void* const* bases_host, int nb) {
  using namespace proj;
  if (nb > kMaxOutMaps) return MUX_OK;
  OutMaps* o = out_maps_find(out_bases_dev, N);
  if (o && o->n == nb) {
    bool same = true;
    for (int r = 0; r < nb; ++r) same = same && o->base[r] == bases_host[r];
    if (same) return MUX_OK;
  }
  o = out_maps_slot(out_bases_dev, N);
  return out_maps_build(*o, out_bases_dev, N, bases_host, nb);
}

namespace proj {

static int make_map(CUtensorMap* m, const void* base, int64_t rows, int cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return MUX_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
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

}  // namespace proj
}  // namespace mux

using namespace mux;

extern "C" int mux_proj_scatter(const uint16_t* X, const uint16_t* W, const uint16_t* bias,
                                int64_t M, int32_t K, int32_t N, const int64_t* row_dst,
                                void* const* out_bases, int32_t num_sms, void* stream) {
  return mux_proj_scatter_dev(X, W, bias, M, nullptr, K, N, row_dst, out_bases, num_sms, stream);
}

extern "C" int mux_proj_scatter_dev(const uint16_t* X, const uint16_t* W, const uint16_t* bias,
                                    int64_t M_max, const int64_t* M_dev, int32_t K, int32_t N,
                                    const int64_t* row_dst, void* const* out_bases,
                                    int32_t num_sms, void* stream) {
  mux_proj_group g{X, W, bias, M_max, M_dev, K, 0, row_dst};
  return mux_proj_scatter_grouped(&g, 1, N, out_bases, num_sms, stream);
}

extern "C" int mux_proj_scatter_grouped(const mux_proj_group* groups, int32_t n_groups,
                                        int32_t N, void* const* out_bases, int32_t num_sms,
                                        void* stream) {
  return mux_proj_scatter_grouped_signal(groups, n_groups, N, out_bases, num_sms, 0, 0, nullptr,
                                         nullptr, nullptr, nullptr, nullptr, nullptr, stream);
}

extern "C" int mux_proj_scatter_grouped_signal(const mux_proj_group* groups, int32_t n_groups,
                                               int32_t N, void* const* out_bases, int32_t num_sms,
                                               int32_t me, int32_t world,
                                               uint64_t* const* flags_peers, uint32_t* sync,
                                               uint64_t* epoch_ctr,
                                               uint64_t* const* e_flags_peers,
                                               uint64_t* e_epoch_ctr, const int32_t* poison,
                                               void* stream) {
  using namespace proj;
  if (world > 0 && (!flags_peers || !sync || !epoch_ctr || world > 32 || me < 0 || me >= world)) {
    set_error("projector signal: need flags, sync and epoch pointers, 0 <= me < world <= 32");
    return MUX_ERR_VALUE;
  }
  if (n_groups < 0 || n_groups > kMaxGroups || N <= 0 || N % BN) {
    set_error("projector: %d groups (max %d), N=%d (need N %% %d == 0)", n_groups, kMaxGroups,
              N, BN);
    return MUX_ERR_VALUE;
  }
  GroupParams P;
  memset(&P, 0, sizeof(P));
  P.N = N;
  P.out_bases = out_bases;
  int64_t tiles = 0;
  const uint16_t* groups_W[kMaxGroups] = {nullptr, nullptr};
  for (int i = 0; i < n_groups; ++i) {
    const mux_proj_group& q = groups[i];
    if (q.K % BK || q.K <= 0 || q.M_max < 0) {
      set_error("projector shape M=%lld K=%d N=%d: need K %% %d == 0 and N %% %d == 0",
                (long long)q.M_max, q.K, N, BK, BN);
      return MUX_ERR_VALUE;
    }
    if (q.M_max == 0) continue;  // nothing to read: drop the group
    const int g = P.n_groups++;
    int st = make_map(&P.ta[g], q.X, q.M_max, q.K, BM);
    if (st) return st;
    st = make_map(&P.tb[g], q.W, N, q.K, BN);
    if (st) return st;
    P.bias[g] = q.bias;
    groups_W[g] = q.W;
    P.row_dst[g] = q.row_dst;
    P.M_dev[g] = q.M_dev;
    P.M_max[g] = q.M_max;
    P.K[g] = q.K;
    tiles += ((q.M_max + BM - 1) / BM) * (N / BN);
  }
  P.flags_peers = flags_peers;
  P.epoch_ctr = epoch_ctr;
  P.ticket = sync;
  P.me = me;
  P.world = world;
  P.e_flags_peers = world > 0 ? e_flags_peers : nullptr;
  P.e_epoch_ctr = e_epoch_ctr;
  P.poison = poison;
  if (P.n_groups == 0) {
    // nothing to compute: still publish the epochs (peers wait for them)
    if (P.e_flags_peers) {
      int st = mux_signal_ex(me, world, e_flags_peers, e_epoch_ctr, 0, stream);
      if (st) return st;
    }
    return world > 0 ? mux_signal(me, world, flags_peers, epoch_ctr, stream) : MUX_OK;
  }
#if MUX_EPI_TMA
  {
    // across GPUs the maps cover the peers' LLM buffers too (TMA stores over
    // NVLink); MUX_EPI_TMA_PEERS=0 keeps the register stores there
    static int peers = -1;
    if (peers < 0) {
      const char* e = getenv("MUX_EPI_TMA_PEERS");
      peers = e ? atoi(e) : 1;
    }
    const int nb = world > 0 ? world : 1;
    const OutMaps* hit = nullptr;
    if ((world <= 0 || peers) && nb <= kMaxOutMaps) {
      int st = out_maps_lookup(out_bases, N, nb, &hit);
      if (st) return st;
    }
    if (hit) {
      P.epi_tma = 1;
      P.n_out = hit->n;
      for (int r = 0; r < hit->n; ++r) {
        P.tout[r] = hit->m[r];
        P.tout_base[r] = hit->base[r];
      }
    }
  }
#endif
  static int pair = -1;  // the CTA-pair (cta_group::2) kernel unless MUX_GEMM_2CTA=0
  if (pair < 0) {
    const char* e = getenv("MUX_GEMM_2CTA");
    pair = e ? atoi(e) : 1;
  }
  if (pair) {
    // B maps with 128-row boxes (each CTA stages half of the 256-column tile)
    for (int g = 0; g < P.n_groups; ++g) {
      int st = make_map(&P.tb[g], groups_W[g], N, P.K[g], 128);
      if (st) return st;
    }
    static bool attr2 = false;
    if (!attr2) {
      MUX_CUDA(cudaFuncSetAttribute(proj_scatter_pair_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2));
      attr2 = true;
    }
    int sms = num_sms;
    if (sms <= 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int64_t tiles2 = 0;
    for (int g = 0; g < P.n_groups; ++g) tiles2 += ((P.M_max[g] + BM2 - 1) / BM2) * (N / BN);
    int pairs = sms / 2;
    if (tiles2 < pairs) pairs = (int)tiles2;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(2 * pairs);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = kSmem2;
    lc.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    MUX_CUDA(cudaLaunchKernelEx(&lc, proj_scatter_pair_kernel, P));
    return MUX_OK;
  }
  static bool attr = false;
  if (!attr) {
    MUX_CUDA(cudaFuncSetAttribute(proj_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmem));
    attr = true;
  }
  int sms = num_sms;
  if (sms <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = (int)(tiles < sms ? tiles : sms);
  proj_scatter_kernel<<<grid, kThreads, kSmem, static_cast<cudaStream_t>(stream)>>>(P);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
