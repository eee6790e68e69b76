// Segment copies: pack, dispatch, return and scatter of the data path (sm_100a).
//
// Every data-plane move of the step is a list of row ranges that are
// contiguous on both sides: a sample's rows are contiguous in the loader
// arena, in the encoder buffer and in its packed LLM sequence.  So pack +
// dispatch (SPEC.md:402 data all-to-all) and return + scatter (SPEC.md:408-416
// restore, "organized as LLM inputs") are one kernel each: a
// persistent grid walks fixed-size chunks of the segment table (chunk map
// built by the planner) and streams bytes with 128-bit loads/stores to a local
// or NVLink-peer destination pointer.  Rows of 1176 B (588 bf16) are only
// 8-byte aligned, so a chunk whose source and destination differ mod 16 uses
// 64-bit accesses; every other chunk uses 128-bit accesses.
//
// The last CTA to finish fences at system scope and publishes `epoch` into the
// completion flag of every peer, so the exchange needs no host round trip.
//
// Failure path: `poison` (nullable device int32, the path's status word) is
// set by a flag wait that timed out (1) or that saw a poisoned peer flag (2).
// A copy launched on a poisoned path moves nothing and publishes its epoch
// with kPoisonBit set, so every peer's wait fails fast instead of copying
// over partial data; waits on a poisoned path return at once.

#include <cstdlib>

#include "mux_common.cuh"

namespace mux {

constexpr int kCopyThreads = 256;
constexpr int kCopyUnroll = 8;  // 8 x 16 B in flight per thread

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_stream2(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_u4(uint4* p, const uint4& v) { *p = v; }

// Block-cooperative copy of n bytes; src, dst and n are multiples of 8.
// After an optional 8-byte head the destination is 16-byte aligned.  If the
// source is then 16-byte aligned too, 128-bit loads/stores stream straight
// through; otherwise (source 8 bytes off, e.g. 1176-byte rows starting at an
// odd row) each lane loads one aligned 16-byte source word and builds its
// destination word from its own high half and its right neighbour's low half
// (warp shuffle), so both sides still move 128 bits per access.
__device__ __forceinline__ void copy_block(char* dst, const char* src, int64_t n) {
  const int tid = threadIdx.x, lane = tid & 31;
  int64_t head = (16 - ((uintptr_t)dst & 15)) & 15;  // 0 or 8
  if (head > n) head = n;
  if (head && tid == 0)
    *reinterpret_cast<uint2*>(dst) = ld_stream2(reinterpret_cast<const uint2*>(src));
  dst += head;
  src += head;
  n -= head;
  const int64_t n16 = n >> 4;
  uint4* d = reinterpret_cast<uint4*>(dst);
  if (((uintptr_t)src & 15) == 0) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    int64_t i = tid;
    for (; i + (kCopyUnroll - 1) * kCopyThreads < n16; i += kCopyUnroll * kCopyThreads) {
      uint4 v[kCopyUnroll];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) v[u] = ld_stream(s + i + u * kCopyThreads);
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) d[i + u * kCopyThreads] = v[u];
    }
    for (; i < n16; i += kCopyThreads) d[i] = ld_stream(s + i);
  } else {
    // source word A[k] = 16 aligned bytes at src - 8 + 16k; dst word k takes
    // A[k].hi and A[k+1].lo.  Warps cover contiguous k so lane+1 holds A[k+1].
    const uint4* A = reinterpret_cast<const uint4*>(src - 8);
    constexpr int U = 4;
    for (int64_t base = 0; base < n16; base += U * kCopyThreads) {
      uint4 v[U];
      uint2 extra[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = base + u * kCopyThreads + tid;
        // A[k] for k < n16 is fully inside the source (its low half is the
        // previous dst word's tail); only the low half of A[n16] is read.
        v[u] = k < n16 ? ld_stream(A + k) : make_uint4(0, 0, 0, 0);
        extra[u] = make_uint2(0, 0);
        if (lane == 31 && k + 1 <= n16)
          extra[u] = ld_stream2(reinterpret_cast<const uint2*>(A + k + 1));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = base + u * kCopyThreads + tid;
        uint32_t nx = __shfl_down_sync(MUX_FULL, v[u].x, 1);
        uint32_t ny = __shfl_down_sync(MUX_FULL, v[u].y, 1);
        if (lane == 31) {
          nx = extra[u].x;
          ny = extra[u].y;
        } else if (k + 1 == n16) {  // neighbour is past the end: A[n16].lo
          const uint2 t = ld_stream2(reinterpret_cast<const uint2*>(A + k + 1));
          nx = t.x;
          ny = t.y;
        }
        if (k < n16) st_u4(d + k, make_uint4(v[u].z, v[u].w, nx, ny));
      }
    }
  }
  const int64_t done = n16 << 4;
  if (done < n && tid == 0)
    *reinterpret_cast<uint2*>(dst + done) =
        ld_stream2(reinterpret_cast<const uint2*>(src + done));
}

struct SegArgs {
  const int64_t* hdr_chunks;  // total chunks
  const int64_t* hdr_segs;    // number of segments
  const int64_t *chunk0, *src_row, *dst_row, *rows;
  const int32_t *group, *rank;
  int64_t chunk_bytes;
  int32_t row_bytes[MUX_N_GROUPS];
  int32_t per_group_dst;  // dispatch: dst index = rank*G + group; return: rank
  void* const* src_bases;
  void* const* dst_bases;
  // fused completion signal (optional)
  uint32_t* sync;       // [0] chunk counter, [1] CTAs done (zero between launches)
  uint64_t* const* flags_peers;
  uint64_t* epoch_ctr;  // device counter: epoch = ++*epoch_ctr (graph-replay safe)
  int32_t me, world;
  int32_t skip_rank;    // segments addressed to this rank are not copied (-1: none)
  int32_t grab;         // chunks per grab (0: adaptive)
  int32_t tail_mult;    // multi-chunk grabs drop to one chunk for the last
                        // tail_mult * grid * grab chunks (0: never)
  const int32_t* poison;  // status word: nonzero = step poisoned, copy nothing
};

// Work distribution is dynamic: CTAs grab chunks (1 for a local copy, kGrab
// for a cross-GPU exchange) from a device counter (the next grab is fetched
// while the current one copies), so
// CTAs that start late — e.g. next to the side-stream planner — take less.
// Each grab locates its first segment by binary search over the chunk prefix
// (staged in shared memory when it fits) and walks forward.
constexpr int kGrab = 4;

__global__ void __launch_bounds__(kCopyThreads) segcopy_kernel(SegArgs a, int smem_segs) {
  extern __shared__ int32_t s_c0[];
  __shared__ uint32_t s_grab[2];
  __shared__ bool s_last;
  const bool poisoned = a.poison && *(volatile const int32_t*)a.poison != 0;
  const int64_t nchunks = poisoned ? 0 : *a.hdr_chunks;
  const int nseg = poisoned ? 0 : (int)*a.hdr_segs;
  const bool staged = nseg < smem_segs;
  if (staged)
    for (int i = threadIdx.x; i <= nseg; i += blockDim.x) s_c0[i] = (int32_t)a.chunk0[i];
  // grab size (measured): one chunk per grab for a local copy —
  // 1184 CTAs share HBM, so a CTA moves only ~5 GB/s and a 4-chunk grab left a
  // ~45 us tail (target-1: 0.171 -> 0.153 ms); kGrab for a cross-GPU exchange,
  // where consecutive chunks to one peer keep NVLink efficient (cfg5 at 4 GPUs:
  // 484 vs 438 M tok/s).  MUX_COPY_GRAB overrides.
  // Near the end multi-chunk grabs shrink to one chunk, so the last CTAs do
  // not leave a tail of up to `grab` chunks each (MUX_COPY_TAIL).
  const uint32_t grab = a.grab > 0 ? (uint32_t)a.grab : (a.flags_peers ? kGrab : 1u);
  const int64_t tail = (int64_t)a.tail_mult * gridDim.x * grab;
  __shared__ uint32_t s_n[2];
  if (threadIdx.x == 0) {
    s_n[0] = grab;
    s_grab[0] = atomicAdd(&a.sync[0], grab);
  }
  __syncthreads();
  auto c0 = [&](int s) -> int64_t { return staged ? s_c0[s] : a.chunk0[s]; };
  for (int buf = 0;; buf ^= 1) {
    const int64_t c_begin = s_grab[buf];
    if (c_begin >= nchunks) break;
    const uint32_t n_this = s_n[buf];
    if (threadIdx.x == 0) {
      const uint32_t gn = nchunks - c_begin <= tail ? 1u : grab;
      s_n[buf ^ 1] = gn;
      s_grab[buf ^ 1] = atomicAdd(&a.sync[0], gn);
    }
    const int64_t c_end = c_begin + n_this < nchunks ? c_begin + n_this : nchunks;
    int lo = 0, hi = nseg - 1;  // last segment with c0 <= c_begin
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (c0(mid) <= c_begin) lo = mid;
      else hi = mid - 1;
    }
    int s = lo;
    int64_t next = c0(s + 1);
    for (int64_t c = c_begin; c < c_end; ++c) {
      while (c >= next) next = c0(++s + 1);
      if (a.rank[s] == a.skip_rank) continue;
      const int g = a.group[s];
      const int64_t rb = a.row_bytes[g];
      const int64_t lo_b = (c - c0(s)) * a.chunk_bytes;
      const int64_t seg = a.rows[s] * rb;
      const int64_t n = seg - lo_b < a.chunk_bytes ? seg - lo_b : a.chunk_bytes;
      const char* src = static_cast<const char*>(a.src_bases[g]) + a.src_row[s] * rb + lo_b;
      const int di = a.per_group_dst ? a.rank[s] * MUX_N_GROUPS + g : a.rank[s];
      char* dst = static_cast<char*>(a.dst_bases[di]) + a.dst_row[s] * rb + lo_b;
      copy_block(dst, src, n);
    }
    __syncthreads();
  }
  // completion: the last CTA re-arms the counters and, for an exchange, fences
  // at system scope and publishes the next epoch to every peer
  if (a.flags_peers) __threadfence_system();  // this thread's peer stores first
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&a.sync[1], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last || threadIdx.x >= 32) return;
  if (threadIdx.x == 0) {
    a.sync[0] = 0;
    a.sync[1] = 0;
  }
  if (a.flags_peers) {
    const uint64_t e = *a.epoch_ctr + 1;
    __syncwarp();
    if (threadIdx.x == 0) *a.epoch_ctr = e;
    __threadfence_system();
    const uint64_t v = poisoned ? (e | kPoisonBit) : e;
    if (threadIdx.x < a.world) {
      uint64_t* f = a.flags_peers[threadIdx.x] + a.me;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
    }
  }
}

// Segment copy through the TMA engine (return / gradient tables whose rows are
// 16-byte multiples; the default for copies without a completion signal, i.e.
// one GPU; MUX_COPY_BULK=0/1 forces it off/on): one thread per CTA grabs chunks from the
// same counter and streams each global -> shared -> global (local or NVLink
// peer) through a ring of kSegBulkBufs 32 KiB buffers, loads running ahead of
// the stores.  Same work units, skip rank, poison and completion signal as
// segcopy_kernel.
constexpr int kSegBulkBufs = 3;

__device__ __forceinline__ bool seg_chunk(const SegArgs& a, int64_t c, int nseg, char*& d,
                                          const char*& s, int64_t& n) {
  int lo = 0, hi = nseg - 1;  // last segment with chunk0 <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.chunk0[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  const int sg = lo;
  if (a.rank[sg] == a.skip_rank) return false;
  const int g = a.group[sg];
  const int64_t rb = a.row_bytes[g];
  const int64_t lo_b = (c - a.chunk0[sg]) * a.chunk_bytes;
  const int64_t seg = a.rows[sg] * rb;
  n = seg - lo_b < a.chunk_bytes ? seg - lo_b : a.chunk_bytes;
  s = static_cast<const char*>(a.src_bases[g]) + a.src_row[sg] * rb + lo_b;
  const int di = a.per_group_dst ? a.rank[sg] * MUX_N_GROUPS + g : a.rank[sg];
  d = static_cast<char*>(a.dst_bases[di]) + a.dst_row[sg] * rb + lo_b;
  return n > 0;
}

__global__ void __launch_bounds__(32) segcopy_bulk_kernel(SegArgs a) {
  extern __shared__ __align__(128) uint8_t seg_bulk_smem[];
  __shared__ uint64_t bar[kSegBulkBufs];
  if (threadIdx.x != 0) return;
  const bool poisoned = a.poison && *(volatile const int32_t*)a.poison != 0;
  const int64_t nchunks = poisoned ? 0 : *a.hdr_chunks;
  const int nseg = poisoned ? 0 : (int)*a.hdr_segs;
  for (int b = 0; b < kSegBulkBufs; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar[b])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  int64_t chunk[kSegBulkBufs];
  char* dst[kSegBulkBufs];
  int32_t len[kSegBulkBufs];
  // issue the load of the next grabbed chunk into buffer b (len 0: nothing to copy)
  auto load = [&](int b) {
    const int64_t c = (int64_t)atomicAdd(&a.sync[0], 1u);
    chunk[b] = c;
    len[b] = 0;
    const char* s = nullptr;
    int64_t n = 0;
    if (c < nchunks && seg_chunk(a, c, nseg, dst[b], s, n)) len[b] = (int32_t)n;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(seg_bulk_smem + b * kDefaultChunkBytes);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[b]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                 "r"((uint32_t)len[b])
                 : "memory");
    if (len[b])
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(sb),
          "l"(s), "r"((uint32_t)len[b]), "r"(mb)
          : "memory");
  };
  uint32_t phase[kSegBulkBufs] = {0, 0, 0};
  for (int b = 0; b < kSegBulkBufs - 1; ++b) load(b);
  for (int j = 0;; ++j) {
    const int b = j % kSegBulkBufs;
    const int nb = (j + kSegBulkBufs - 1) % kSegBulkBufs;
    if (chunk[b] >= nchunks) break;  // grabs are increasing: nothing further either
    // buffer nb is reused for the next grab: its previous store must have read it
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    load(nb);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[b]);
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(mb),
        "r"(phase[b])
        : "memory");
    phase[b] ^= 1;
    if (len[b]) {
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(seg_bulk_smem + b * kDefaultChunkBytes);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst[b]),
                   "r"(sb), "r"((uint32_t)len[b])
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (a.flags_peers) __threadfence_system();
  const bool last = atomicAdd(&a.sync[1], 1u) == gridDim.x - 1;
  if (!last) return;
  a.sync[0] = 0;
  a.sync[1] = 0;
  if (a.flags_peers) {
    const uint64_t e = *a.epoch_ctr + 1;
    *a.epoch_ctr = e;
    __threadfence_system();
    const uint64_t v = poisoned ? (e | kPoisonBit) : e;
    for (int r = 0; r < a.world; ++r) {
      uint64_t* f = a.flags_peers[r] + a.me;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
    }
  }
}

// One contiguous byte range (probe / utility): grid-stride 32 KiB blocks.
__global__ void __launch_bounds__(kCopyThreads) copy_bytes_kernel(char* dst, const char* src,
                                                                  int64_t n) {
  const int64_t CH = kDefaultChunkBytes;
  for (int64_t lo = (int64_t)blockIdx.x * CH; lo < n; lo += (int64_t)gridDim.x * CH)
    copy_block(dst + lo, src + lo, n - lo < CH ? n - lo : CH);
}

// ---------------------------------------------------------------------------
// Multi-range copy (NVLink probe, copy-engine A/B): n ranges, 32 KiB chunks
// dealt round-robin over the ranges so every destination is written at once.
// mode 0: SM loads/stores (copy_block); mode 1: TMA bulk copies — each CTA
// streams its chunks global -> shared (cp.async.bulk, mbarrier) -> global
// (cp.async.bulk.global.shared::cta) through a ring of kBulkBufs buffers.
// ---------------------------------------------------------------------------
constexpr int kBulkChunk = 32768, kBulkBufs = 3;

struct RangeArgs {
  int n;
  void* const* dst;
  const void* const* src;
  const int64_t* bytes;
  int64_t max_chunks;  // chunks of the longest range
};

__device__ __forceinline__ bool range_chunk(const RangeArgs& a, int64_t c, char*& d, const char*& s,
                                            int64_t& len) {
  const int r = (int)(c % a.n);
  const int64_t k = c / a.n;
  const int64_t lo = k * kBulkChunk, b = a.bytes[r];
  if (lo >= b) return false;
  len = b - lo < kBulkChunk ? b - lo : kBulkChunk;
  d = static_cast<char*>(a.dst[r]) + lo;
  s = static_cast<const char*>(a.src[r]) + lo;
  return true;
}

__global__ void __launch_bounds__(kCopyThreads) ranges_sm_kernel(RangeArgs a) {
  const int64_t total = a.max_chunks * a.n;
  for (int64_t c = blockIdx.x; c < total; c += gridDim.x) {
    char* d;
    const char* s;
    int64_t len;
    if (range_chunk(a, c, d, s, len)) copy_block(d, s, len);
  }
}

__global__ void __launch_bounds__(32) ranges_bulk_kernel(RangeArgs a) {
  extern __shared__ __align__(128) uint8_t bulk_smem[];
  __shared__ uint64_t bar[kBulkBufs];
  if (threadIdx.x != 0) return;
  const int64_t total = a.max_chunks * a.n;
  // this CTA's chunks: c = blockIdx.x + j * gridDim.x, j = 0, 1, ...
  for (int b = 0; b < kBulkBufs; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar[b])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto load = [&](int64_t j) {  // issue the load of this CTA's chunk j into buffer j % NB
    const int b = (int)(j % kBulkBufs);
    char* d;
    const char* s;
    int64_t len = 0;
    const int64_t c = blockIdx.x + j * gridDim.x;
    if (c >= total || !range_chunk(a, c, d, s, len)) len = 0;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bulk_smem + b * kBulkChunk);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[b]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                 "r"((uint32_t)len)
                 : "memory");
    if (len)
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(sb),
          "l"(s), "r"((uint32_t)len), "r"(mb)
          : "memory");
  };
  const int64_t mine = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (int64_t j = 0; j < kBulkBufs - 1 && j < mine; ++j) load(j);
  for (int64_t j = 0; j < mine; ++j) {
    if (j + kBulkBufs - 1 < mine) {
      // buffer (j - 1) % NB is reused: the store of chunk j-1 must have read it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(j + kBulkBufs - 1);
    }
    const int b = (int)(j % kBulkBufs);
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&bar[b]);
    const uint32_t par = (uint32_t)((j / kBulkBufs) & 1);
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(mb),
        "r"(par)
        : "memory");
    char* d;
    const char* s;
    int64_t len;
    const int64_t c = blockIdx.x + j * gridDim.x;
    if (range_chunk(a, c, d, s, len)) {
      const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bulk_smem + b * kBulkChunk);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(sb),
                   "r"((uint32_t)len)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void signal_kernel(int me, int world, uint64_t* const* flags_peers,
                              uint64_t* epoch_ctr, int fence) {
  const int r = threadIdx.x;
  const uint64_t e = *epoch_ctr + 1;
  __syncwarp();
  if (r == 0) *epoch_ctr = e;
  // fence = 0: a pure permission ("my buffer may be overwritten") after
  // kernels that only READ it; stream order already completed those reads
  if (fence) __threadfence_system();
  if (r < world) {
    uint64_t* f = flags_peers[r] + me;
    if (fence)
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
    else
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
  }
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void wait_kernel(int world, const uint64_t* flags, const uint64_t* epoch_ctr,
                            uint64_t target, int64_t timeout_ns, int32_t* err) {
  const int r = threadIdx.x;
  if (r >= world) return;
  if (*(volatile int32_t*)err != 0) return;  // poisoned path: fail fast
  const uint64_t epoch = epoch_ctr ? *epoch_ctr : target;
  const uint64_t t0 = global_ns();
  for (;;) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + r) : "memory");
    if (v & kPoisonBit) {  // the peer's step was poisoned: so is ours
      atomicCAS(err, 0, 2);
      break;
    }
    if (v >= epoch) break;
    if ((int64_t)(global_ns() - t0) > timeout_ns) {
      atomicExch(err, 1);
      break;
    }
    __nanosleep(128);
  }
}

// ---------------------------------------------------------------------------
// encoder stand-in E(id, t, c): a deterministic hash mapped to a finite bf16
// in +-[0.5, 2).  oracle/dataplane.py:standin restates it bit for bit.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint32_t standin_bits(uint32_t row_seed, uint32_t c) {
  const uint32_t h = mix32(row_seed ^ (c * 0x85ebca77u));
  return ((h >> 31) << 15) | ((126u + ((h >> 7) & 1u)) << 7) | (h & 0x7fu);
}

__global__ void __launch_bounds__(256) standin_kernel(Plan p, int S, int me, int group,
                                                     const int64_t* ids, const int32_t* lens,
                                                     int width, uint16_t* out, int lssp_G) {
  for (int i = blockIdx.y; i < S; i += gridDim.y) {
    if (p.group[i] != group) continue;
    // rows of sample i this rank encodes: tokens [t0, t0 + L) at rows r0..
    int t0 = 0, L = lens[i];
    int64_t r0;
    if (lssp_G > 0) {  // LSSP: DP samples whole at home, SP shard k on member k
      const int st = p.lssp_state[i], e = p.enc[i];
      if (st == 0) {
        if (e != me) continue;
        r0 = p.lssp_row[(int64_t)i * MUX_LSSP_MAX];
      } else if (st == 1) {
        const int k = me - (e - e % lssp_G);
        if (k < 0 || k >= lssp_G) continue;
        const int b = L / lssp_G, rem = L % lssp_G;
        t0 = k * b + (k < rem ? k : rem);
        L = b + (k < rem ? 1 : 0);
        r0 = p.lssp_row[(int64_t)i * MUX_LSSP_MAX + k];
      } else {
        continue;
      }
    } else {
      if (p.enc[i] != me) continue;
      r0 = p.enc_off[i];
    }
    const int64_t id = ids[i];
    const uint32_t sseed = mix32((uint32_t)id ^ mix32((uint32_t)((uint64_t)id >> 32) + 0x632be59bu));
    const int nv = width / 8;
    for (int j = blockIdx.x; j < L; j += gridDim.x) {
      const int t = t0 + j;
      const uint32_t rs = mix32(sseed + (uint32_t)t * 0x9e3779b9u);
      uint4* row = reinterpret_cast<uint4*>(out + (r0 + j) * width);
      for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        const uint32_t c = v * 8;
        uint4 w;
        w.x = standin_bits(rs, c) | (standin_bits(rs, c + 1) << 16);
        w.y = standin_bits(rs, c + 2) | (standin_bits(rs, c + 3) << 16);
        w.z = standin_bits(rs, c + 4) | (standin_bits(rs, c + 5) << 16);
        w.w = standin_bits(rs, c + 6) | (standin_bits(rs, c + 7) << 16);
        row[v] = w;
      }
    }
  }
}

// row_dst[src row] = (dst rank << 40) | dst row of every return piece of
// `group` (group < 0: every group, group g's map at row_dst + g * n_rows).
__global__ void return_rows_kernel(Plan p, int group, int64_t* row_dst, int64_t n_rows) {
  const int64_t npieces = p.hdr[MUX_H_N_RETURN];
  for (int64_t s = blockIdx.x; s < npieces; s += gridDim.x) {
    if (group >= 0 && p.rgroup[s] != group) continue;
    int64_t* rd = group >= 0 ? row_dst : row_dst + (int64_t)p.rgroup[s] * n_rows;
    const int64_t src = p.rsrc[s], dst = p.rdst[s], n = p.rrows[s];
    const int64_t tag = (int64_t)p.rrank[s] << 40;
    for (int64_t t = threadIdx.x; t < n; t += blockDim.x)
      if (src + t < n_rows) rd[src + t] = tag | (dst + t);
  }
}

// Text rows of the packed LLM input: one warp per row, the embedding row of
// the token id gathered with 128-bit loads.
__global__ void __launch_bounds__(256) text_embed_kernel(Plan p, const int32_t* tokens,
                                                         const uint16_t* table, int64_t vocab,
                                                         int d, uint16_t* out, int32_t* err) {
  const int64_t nseg = p.hdr[MUX_H_N_TEXT], rows = p.hdr[MUX_H_TEXT_ROWS];
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nv = d / 8;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    int64_t lo = 0, hi = nseg - 1;  // last segment with trow0 <= r
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (p.trow0[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int64_t t = r - p.trow0[lo];
    const int32_t tok = tokens[p.tsrc[lo] + t];
    if (tok < 0 || tok >= vocab) {
      if (lane == 0) atomicAdd(err, 1);
      continue;
    }
    const uint4* src = reinterpret_cast<const uint4*>(table + (int64_t)tok * d);
    uint4* dst = reinterpret_cast<uint4*>(out + (p.tdst[lo] + t) * d);
#pragma unroll 4
    for (int v = lane; v < nv; v += 32) dst[v] = __ldg(src + v);
  }
}

// Staged projector return: row_dst of the owner's staging rows of `group`.
__global__ void stage_rows_kernel(Plan p, const int32_t* lens, int S, int me, int group,
                                  int64_t* row_dst, int64_t n_rows) {
  for (int i = blockIdx.x; i < S; i += gridDim.x) {
    if (p.origin[i] != me || p.group[i] != group || p.enc[i] < 0) continue;
    const int64_t s0 = p.stage_off[i], l0 = p.llm_row[i];
    const int64_t tag = (int64_t)me << 40;
    for (int64_t t = threadIdx.x; t < lens[i]; t += blockDim.x)
      if (s0 + t < n_rows) row_dst[s0 + t] = tag | (l0 + t);
  }
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace mux

using namespace mux;

extern "C" int mux_segcopy(const mux_plan_cfg* cfg, const void* plan, int32_t which,
                           void* const* src_bases, void* const* dst_bases, int32_t grid_ctas,
                           uint32_t* sync, void* stream) {
  return mux_segcopy_signal(cfg, plan, which, src_bases, dst_bases, grid_ctas, nullptr, sync,
                            nullptr, stream);
}

extern "C" int mux_segcopy_signal(const mux_plan_cfg* cfg, const void* plan, int32_t which,
                                  void* const* src_bases, void* const* dst_bases,
                                  int32_t grid_ctas, uint64_t* const* flags_peers,
                                  uint32_t* sync, uint64_t* epoch_ctr, void* stream) {
  return mux_segcopy_ex(cfg, plan, which, src_bases, dst_bases, grid_ctas, -1, flags_peers, sync,
                        epoch_ctr, nullptr, stream);
}

extern "C" int mux_segcopy_ex(const mux_plan_cfg* cfg, const void* plan, int32_t which,
                              void* const* src_bases, void* const* dst_bases, int32_t grid_ctas,
                              int32_t skip_rank, uint64_t* const* flags_peers, uint32_t* sync,
                              uint64_t* epoch_ctr, const int32_t* poison, void* stream) {
  mux_plan_layout L;
  int st = mux_plan_layout_of(cfg, &L);
  if (st) return st;
  Plan p = make_plan_const(plan, L);
  SegArgs a;
  if (which < 0 || which > 2) {
    set_error("segment table %d: 0 dispatch, 1 return, 2 gradient return", which);
    return MUX_ERR_VALUE;
  }
  const bool ret = which != 0;
  const bool grad = which == 2;
  a.hdr_chunks = p.hdr + (grad ? MUX_H_GRAD_CHUNKS : ret ? MUX_H_RETURN_CHUNKS
                                                         : MUX_H_DISPATCH_CHUNKS);
  a.hdr_segs = p.hdr + (grad ? MUX_H_N_GRAD : ret ? MUX_H_N_RETURN : MUX_H_N_DISPATCH);
  a.chunk0 = grad ? p.gchunk0 : ret ? p.rchunk0 : p.dchunk0;
  a.src_row = grad ? p.gsrc : ret ? p.rsrc : p.dsrc;
  a.dst_row = grad ? p.gdst : ret ? p.rdst : p.ddst;
  a.rows = grad ? p.grows : ret ? p.rrows : p.drows;
  a.group = grad ? p.ggroup : ret ? p.rgroup : p.dgroup;
  a.rank = grad ? p.grank : ret ? p.rrank : p.drank;
  a.chunk_bytes = cfg->chunk_bytes > 0 ? cfg->chunk_bytes : kDefaultChunkBytes;
  for (int g = 0; g < MUX_N_GROUPS; ++g)
    a.row_bytes[g] = grad ? (cfg->row_bytes_grad[g] > 0 ? cfg->row_bytes_grad[g]
                                                        : cfg->row_bytes_ret[g])
                          : ret ? cfg->row_bytes_ret[g] : cfg->row_bytes_in[g];
  a.per_group_dst = (!ret || grad || cfg->ret_mode == MUX_RET_STAGED) ? 1 : 0;
  a.src_bases = src_bases;
  a.dst_bases = dst_bases;
  a.flags_peers = flags_peers;
  a.sync = sync;
  a.epoch_ctr = epoch_ctr;
  a.me = cfg->me;
  a.world = cfg->world;
  a.skip_rank = skip_rank;
  a.poison = poison;
  static int grab = -1;  // MUX_COPY_GRAB (tuning; 0 = adaptive)
  if (grab < 0) {
    const char* e = getenv("MUX_COPY_GRAB");
    grab = e ? atoi(e) : 0;
  }
  a.grab = grab;
  // MUX_COPY_TAIL (default 1, measured: cfg5 at 2 GPUs 294 vs 279 M tok/s; at 4
  // GPUs 448-454 vs 448-457, 2 and 4 were slower there)
  static int tail_mult = -1;
  if (tail_mult < 0) {
    const char* e = getenv("MUX_COPY_TAIL");
    tail_mult = e ? atoi(e) : 1;
  }
  a.tail_mult = tail_mult;
  if (!sync || (flags_peers && !epoch_ctr)) {
    set_error("segment copy needs its sync counters (and an epoch counter to signal)");
    return MUX_ERR_VALUE;
  }
  // grid_ctas < 0: "co-resident" launch of -grid_ctas CTAs with no shared
  // memory, so the copy can run beside a kernel that holds the SMs' shared
  // memory (the projector GEMM); otherwise the chunk prefix is staged in
  // shared memory when the segment bound is small.
  const bool lean = grid_ctas < 0;
  // MUX_COPY_BULK: TMA-engine copies for 16-byte-multiple rows.  Default: only
  // without a completion signal (one GPU / a local copy), where it measured +3% on
  // target-1; across GPUs its NVLink rate measured lower (392 vs 427 GB/s at 4).
  static int bulk_env = -2;
  if (bulk_env == -2) {
    const char* e = getenv("MUX_COPY_BULK");
    bulk_env = e ? atoi(e) : -1;
  }
  const bool bulk = bulk_env < 0 ? flags_peers == nullptr : bulk_env != 0;
  if (bulk && !lean && ret && a.chunk_bytes <= kDefaultChunkBytes && a.chunk_bytes % 16 == 0 &&
      a.row_bytes[0] % 16 == 0 && a.row_bytes[1] % 16 == 0) {
    static bool attr = false;
    if (!attr) {
      MUX_CUDA(cudaFuncSetAttribute(segcopy_bulk_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSegBulkBufs * kDefaultChunkBytes));
      attr = true;
    }
    const int bgrid = grid_ctas > 0 ? grid_ctas : num_sms() * 2;
    segcopy_bulk_kernel<<<bgrid, 32, kSegBulkBufs * kDefaultChunkBytes,
                          static_cast<cudaStream_t>(stream)>>>(a);
    MUX_CUDA(cudaGetLastError());
    return MUX_OK;
  }
  const int grid = lean ? -grid_ctas : (grid_ctas > 0 ? grid_ctas : num_sms() * 8);
  const int max_segs = ret ? cfg->S * (cfg->sp + 1) + 1 : cfg->S + 1;
  const int smem_segs = !lean && max_segs + 1 <= 4096 ? max_segs + 1 : 0;
  segcopy_kernel<<<grid, kCopyThreads, smem_segs * sizeof(int32_t),
                   static_cast<cudaStream_t>(stream)>>>(a, smem_segs);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_signal(int32_t me, int32_t world, uint64_t* const* flags_peers,
                          uint64_t* epoch_ctr, void* stream) {
  return mux_signal_ex(me, world, flags_peers, epoch_ctr, 1, stream);
}

extern "C" int mux_signal_ex(int32_t me, int32_t world, uint64_t* const* flags_peers,
                             uint64_t* epoch_ctr, int32_t fence, void* stream) {
  signal_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(me, world, flags_peers,
                                                                 epoch_ctr, fence);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_wait(int32_t world, const uint64_t* my_flags, const uint64_t* epoch_ctr,
                        int32_t timeout_ms, int32_t* err_dev, void* stream) {
  wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(world, my_flags, epoch_ctr, 0,
                                                               (int64_t)timeout_ms * 1000000,
                                                               err_dev);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_wait_value(int32_t world, const uint64_t* my_flags, uint64_t target,
                              int32_t timeout_ms, int32_t* err_dev, void* stream) {
  wait_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(world, my_flags, nullptr, target,
                                                               (int64_t)timeout_ms * 1000000,
                                                               err_dev);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_encoder_standin(const mux_plan_cfg* cfg, const void* plan, const int64_t* ids,
                                   const int32_t* lens, int32_t group, int32_t width,
                                   uint16_t* out, void* stream) {
  if (width % 8) {
    set_error("stand-in width %d must be a multiple of 8", width);
    return MUX_ERR_VALUE;
  }
  mux_plan_layout L;
  int st = mux_plan_layout_of(cfg, &L);
  if (st) return st;
  Plan p = make_plan_const(plan, L);
  dim3 grid(64, cfg->S > 0 ? (cfg->S < 1024 ? cfg->S : 1024) : 1);
  standin_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      p, cfg->S, cfg->me, group, ids, lens, width, out, cfg->lssp_sp);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_return_rows(const mux_plan_cfg* cfg, const void* plan, int32_t group,
                               int64_t* row_dst, int64_t n_rows, void* stream) {
  mux_plan_layout L;
  int st = mux_plan_layout_of(cfg, &L);
  if (st) return st;
  Plan p = make_plan_const(plan, L);
  return_rows_kernel<<<256, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, group, row_dst,
                                                                         n_rows);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_text_embed(const mux_plan_cfg* cfg, const void* plan, const int32_t* tokens,
                              const uint16_t* table, int64_t vocab, int32_t d, uint16_t* out,
                              int32_t* err, void* stream) {
  if (!cfg->text_embed || cfg->mode != MUX_MODE_STEP) {
    set_error("mux_text_embed needs a step plan made with text_embed = 1");
    return MUX_ERR_VALUE;
  }
  if (d <= 0 || d % 8 || vocab <= 0 ||
      (((uintptr_t)table | (uintptr_t)out) & 15) != 0) {
    set_error("mux_text_embed: need d %% 8 == 0, vocab > 0, 16-byte aligned table and out");
    return MUX_ERR_VALUE;
  }
  mux_plan_layout L;
  int st = mux_plan_layout_of(cfg, &L);
  if (st) return st;
  Plan p = make_plan_const(plan, L);
  text_embed_kernel<<<num_sms() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      p, tokens, table, vocab, d, out, err);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_copy_bytes(void* dst, const void* src, int64_t n, int32_t grid_ctas,
                              void* stream) {
  if ((((uintptr_t)dst | (uintptr_t)src | (uintptr_t)n) & 7) != 0) {
    set_error("mux_copy_bytes needs 8-byte aligned pointers and size");
    return MUX_ERR_VALUE;
  }
  if (n == 0) return MUX_OK;
  const int grid = grid_ctas > 0 ? grid_ctas : num_sms() * 8;
  copy_bytes_kernel<<<grid, kCopyThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<char*>(dst), static_cast<const char*>(src), n);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_copy_ranges(int32_t n, void* const* dsts, const void* const* srcs,
                               const int64_t* bytes, int64_t max_bytes, int32_t grid_ctas,
                               int32_t mode, void* stream) {
  if (n <= 0 || !dsts || !srcs || !bytes || max_bytes < 0 || (mode != 0 && mode != 1)) {
    set_error("mux_copy_ranges: n > 0, device arrays, max_bytes >= 0, mode 0 (SM) or 1 (TMA)");
    return MUX_ERR_VALUE;
  }
  RangeArgs a{n, dsts, srcs, bytes, (max_bytes + kBulkChunk - 1) / kBulkChunk};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mode == 0) {
    ranges_sm_kernel<<<grid_ctas > 0 ? grid_ctas : num_sms() * 8, kCopyThreads, 0, s>>>(a);
  } else {
    static bool attr = false;
    if (!attr) {
      MUX_CUDA(cudaFuncSetAttribute(ranges_bulk_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kBulkBufs * kBulkChunk));
      attr = true;
    }
    ranges_bulk_kernel<<<grid_ctas > 0 ? grid_ctas : num_sms() * 2, 32, kBulkBufs * kBulkChunk,
                         s>>>(a);
  }
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_memcpy_async(void* dst, const void* src, int64_t n, void* stream) {
  MUX_CUDA(cudaMemcpyAsync(dst, src, (size_t)n, cudaMemcpyDefault,
                           static_cast<cudaStream_t>(stream)));
  return MUX_OK;
}

extern "C" int mux_stage_rows(const mux_plan_cfg* cfg, const void* plan, const int32_t* lens,
                              int32_t group, int64_t* row_dst, int64_t n_rows, void* stream) {
  if (cfg->ret_mode != MUX_RET_STAGED) {
    set_error("mux_stage_rows needs a plan made with ret_mode MUX_RET_STAGED");
    return MUX_ERR_VALUE;
  }
  mux_plan_layout L;
  int st = mux_plan_layout_of(cfg, &L);
  if (st) return st;
  Plan p = make_plan_const(plan, L);
  const int grid = cfg->S > 0 ? (cfg->S < 1024 ? cfg->S : 1024) : 1;
  stage_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(p, lens, cfg->S,
                                                                         cfg->me, group,
                                                                         row_dst, n_rows);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
