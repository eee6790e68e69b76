// Device planner for one step of the encoder<->LLM data path (sm_100a).
//
// K_ffd      one CTA per drawn chunk: bitonic sort by (-len, id, index) and a
//            warp-synchronous first fit over the bins
//            (reference: pkg/src/muxsim/workload.py:240-262).
// K_finalize one CTA: carry spans, global sequence ids, error checks
//            (workload.py:245-248, :269-275), batch slice + replica owner
//            (:265-280, :177-180), Ulysses shard geometry,
//            origin / loader-arena / encoder assignment (LPT or KK;
//            SPEC.md:390-407), encoder order, return pieces and the
//            per-rank segment tables consumed by the copy kernels.
// Everything is integer (or exact double) arithmetic, deterministic and
// identical on every rank, so every rank can plan the whole step locally and
// push its rows without exchanging counts.

#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "mux_common.cuh"

namespace mux {

// --------------------------------------------------------------------------
// layout
// --------------------------------------------------------------------------

static int compute_layout(const mux_plan_cfg& c, mux_plan_layout* L) {
  if (c.S < 0 || c.n_carry < 0 || c.n_carry > c.S || c.n_chunks < 0 || c.n_carry_seqs < 0) {
    set_error("invalid step table sizes");
    return MUX_ERR_VALUE;
  }
  if (c.S > 4096) {
    set_error("step table of %d samples exceeds the device planner limit 4096", c.S);
    return MUX_ERR_VALUE;
  }
  if (c.mode == MUX_MODE_STEP) {
    if (c.world < 1 || c.world > 8 || c.sp < 1 || c.dp < 1 || c.gbs < 0 || c.mbs < 1) {
      set_error("invalid world/dp/sp/gbs/mbs");
      return MUX_ERR_VALUE;
    }
    if ((int64_t)c.gbs * c.sp > 4096) {
      set_error("gbs x sp exceeds the device planner limit 4096");
      return MUX_ERR_VALUE;
    }
  }
  const int64_t S = c.S > 0 ? c.S : 1;
  const int64_t nch = c.n_chunks > 0 ? c.n_chunks : 1;
  const int64_t mseq = max_seq_of(c);
  const int64_t gb = (c.gbs > 0 ? c.gbs : 1) * (c.sp > 0 ? c.sp : 1);
  const int64_t W = (c.world > 0 ? c.world : 1);
  const int64_t R = max_ret_of(c);
  const int64_t MC = c.max_chunks > 0 ? c.max_chunks : 1;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    int64_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L->header = take(8 * MUX_H_SLOTS);
  L->seq = take(4 * S);
  L->off = take(4 * S);
  L->span = take(4 * S);
  L->origin = take(4 * S);
  L->origin_pos = take(4 * S);
  L->group = take(4 * S);
  L->enc = take(4 * S);
  L->arena_off = take(8 * S);
  L->enc_off = take(8 * S);
  L->llm_rank = take(4 * S);
  L->llm_row = take(8 * S);
  L->bin_fill = take(4 * S);
  L->bin_nspan = take(4 * S);
  L->bin_of = take(4 * S);
  L->chunk_nbins = take(4 * nch);
  L->fills = take(4 * mseq);
  L->nspans = take(4 * mseq);
  L->cu = take(4 * (gb + 1));
  L->shard_len = take(4 * gb);
  L->shard_start = take(4 * gb);
  L->row_base = take(8 * gb);
  L->arena_rows = take(8 * W * MUX_N_GROUPS);
  L->recv_rows = take(8 * W * MUX_N_GROUPS);
  L->llm_rows = take(8 * W);
  L->order = take(4 * S);
  L->scratch_a = take(4 * S);
  L->scratch_b = take(4 * S);
  L->dseg_src_row = take(8 * S);
  L->dseg_dst_row = take(8 * S);
  L->dseg_rows = take(8 * S);
  L->dseg_group = take(4 * S);
  L->dseg_dst_rank = take(4 * S);
  L->dseg_chunk0 = take(8 * (S + 1));
  L->dchunk_seg = take(4 * MC);
  L->rseg_src_row = take(8 * R);
  L->rseg_dst_row = take(8 * R);
  L->rseg_rows = take(8 * R);
  L->rseg_group = take(4 * R);
  L->rseg_dst_rank = take(4 * R);
  L->rseg_chunk0 = take(8 * (R + 1));
  L->rchunk_seg = take(4 * MC);
  L->total = o;
  return MUX_OK;
}

template <typename T>
static T* at(void* base, int64_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

Plan make_plan(void* b, const mux_plan_layout& L) {
  Plan p;
  p.hdr = at<int64_t>(b, L.header);
  p.seq = at<int32_t>(b, L.seq);
  p.off = at<int32_t>(b, L.off);
  p.span = at<int32_t>(b, L.span);
  p.origin = at<int32_t>(b, L.origin);
  p.origin_pos = at<int32_t>(b, L.origin_pos);
  p.group = at<int32_t>(b, L.group);
  p.enc = at<int32_t>(b, L.enc);
  p.arena_off = at<int64_t>(b, L.arena_off);
  p.enc_off = at<int64_t>(b, L.enc_off);
  p.llm_rank = at<int32_t>(b, L.llm_rank);
  p.llm_row = at<int64_t>(b, L.llm_row);
  p.bin_fill = at<int32_t>(b, L.bin_fill);
  p.bin_nspan = at<int32_t>(b, L.bin_nspan);
  p.bin_of = at<int32_t>(b, L.bin_of);
  p.chunk_nbins = at<int32_t>(b, L.chunk_nbins);
  p.fills = at<int32_t>(b, L.fills);
  p.nspans = at<int32_t>(b, L.nspans);
  p.cu = at<int32_t>(b, L.cu);
  p.shard_len = at<int32_t>(b, L.shard_len);
  p.shard_start = at<int32_t>(b, L.shard_start);
  p.row_base = at<int64_t>(b, L.row_base);
  p.arena_rows = at<int64_t>(b, L.arena_rows);
  p.recv_rows = at<int64_t>(b, L.recv_rows);
  p.llm_rows = at<int64_t>(b, L.llm_rows);
  p.order = at<int32_t>(b, L.order);
  p.scratch_a = at<int32_t>(b, L.scratch_a);
  p.scratch_b = at<int32_t>(b, L.scratch_b);
  p.dsrc = at<int64_t>(b, L.dseg_src_row);
  p.ddst = at<int64_t>(b, L.dseg_dst_row);
  p.drows = at<int64_t>(b, L.dseg_rows);
  p.dgroup = at<int32_t>(b, L.dseg_group);
  p.drank = at<int32_t>(b, L.dseg_dst_rank);
  p.dchunk0 = at<int64_t>(b, L.dseg_chunk0);
  p.dchunk_seg = at<int32_t>(b, L.dchunk_seg);
  p.rsrc = at<int64_t>(b, L.rseg_src_row);
  p.rdst = at<int64_t>(b, L.rseg_dst_row);
  p.rrows = at<int64_t>(b, L.rseg_rows);
  p.rgroup = at<int32_t>(b, L.rseg_group);
  p.rrank = at<int32_t>(b, L.rseg_dst_rank);
  p.rchunk0 = at<int64_t>(b, L.rseg_chunk0);
  p.rchunk_seg = at<int32_t>(b, L.rchunk_seg);
  return p;
}

Plan make_plan_const(const void* b, const mux_plan_layout& L) {
  return make_plan(const_cast<void*>(b), L);
}

// --------------------------------------------------------------------------
// K_ffd: first-fit decreasing of one chunk
// --------------------------------------------------------------------------

constexpr int kFfdThreads = 512;
constexpr int kRegSlots = 8;  // bins kept in registers: 32 lanes x 8 = 256

struct FfdKey {
  const int32_t* len;
  const int64_t* id;
  int n;
  // (-len, id, index) ascending; padding (>= n) last.  Stable == index tie.
  __device__ bool operator()(int a, int b) const {
    if (a >= n) return false;
    if (b >= n) return true;
    if (len[a] != len[b]) return len[a] > len[b];
    if (id[a] != id[b]) return id[a] < id[b];
    return a < b;
  }
};

__global__ void __launch_bounds__(kFfdThreads) ffd_kernel(mux_plan_cfg cfg, const int32_t* lens,
                                                          const int64_t* ids,
                                                          const int32_t* chunk_off, Plan p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t s_warp[33];
  const int c = blockIdx.x;
  const int lo = chunk_off[c], n = chunk_off[c + 1] - lo;
  const int npad = next_pow2(n > 0 ? n : 1);
  int64_t* s_id = reinterpret_cast<int64_t*>(smem);
  int32_t* s_len = reinterpret_cast<int32_t*>(s_id + npad);
  int32_t* s_ord = s_len + npad;
  int32_t* s_fill = s_ord + npad;   // smem first-fit path only
  int32_t* s_nsp = s_fill + npad;
  const int cap = cfg.capacity;

  int64_t my_total = 0;
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    if (i < n) {
      const int L = lens[lo + i];
      s_len[i] = L;
      s_id[i] = ids[lo + i];
      my_total += L;
      if (L > cap)  // first offender in table order wins (workload.py:245-248)
        atomicMin(reinterpret_cast<unsigned long long*>(&p.hdr[MUX_H_ERR_INDEX]),
                  (unsigned long long)(lo + i));
    }
    s_ord[i] = i;
  }
  int64_t total;
  block_excl_scan(my_total, &total, s_warp);
  bitonic_sort(s_ord, npad, FfdKey{s_len, s_id, n});

  // FF never leaves two bins at most half full, so #bins <= 2*total/cap + 1.
  const int64_t bound = cap > 0 ? 2 * total / cap + 2 : n;
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int nb = 0;
  if (bound <= 32 * kRegSlots) {
    int fill[kRegSlots], nsp[kRegSlots];
#pragma unroll
    for (int s = 0; s < kRegSlots; ++s) fill[s] = nsp[s] = 0;
    int nxt_i = n > 0 ? s_ord[0] : 0;
    int nxt_L = n > 0 ? s_len[nxt_i] : 0;
    for (int q = 0; q < n; ++q) {
      const int i = nxt_i, L = nxt_L;
      if (q + 1 < n) {
        nxt_i = s_ord[q + 1];
        nxt_L = s_len[nxt_i];
      }
      int cand = INT_MAX;
#pragma unroll
      for (int s = kRegSlots - 1; s >= 0; --s) {
        const int b = s * 32 + lane;
        if (b < nb && fill[s] + L <= cap) cand = b;
      }
      int best = __reduce_min_sync(MUX_FULL, cand);
      if (best == INT_MAX) best = nb++;
      if (lane == (best & 31)) {
        const int slot = best >> 5;
        int fo = 0, so = 0;
#pragma unroll
        for (int s = 0; s < kRegSlots; ++s)
          if (s == slot) {
            fo = fill[s];
            so = nsp[s];
            fill[s] = fo + L;
            nsp[s] = so + 1;
          }
        p.bin_of[lo + i] = best;
        p.off[lo + i] = fo;
        p.span[lo + i] = so;
      }
    }
#pragma unroll
    for (int s = 0; s < kRegSlots; ++s) {
      const int b = s * 32 + lane;
      if (b < nb) {
        p.bin_fill[lo + b] = fill[s];
        p.bin_nspan[lo + b] = nsp[s];
      }
    }
  } else {
    for (int q = 0; q < n; ++q) {
      const int i = s_ord[q], L = s_len[i];
      int best = -1;
      for (int base = 0; base < nb; base += 32) {
        const int b = base + lane;
        const bool fit = b < nb && s_fill[b] + L <= cap;
        const unsigned bal = __ballot_sync(MUX_FULL, fit);
        if (bal) {
          best = base + __ffs(bal) - 1;
          break;
        }
      }
      if (best < 0) {
        best = nb++;
        if (lane == 0) s_fill[best] = s_nsp[best] = 0;
        __syncwarp();
      }
      if (lane == 0) {
        p.bin_of[lo + i] = best;
        p.off[lo + i] = s_fill[best];
        p.span[lo + i] = s_nsp[best];
        s_fill[best] += L;
        s_nsp[best] += 1;
      }
      __syncwarp();
    }
    for (int b = lane; b < nb; b += 32) {
      p.bin_fill[lo + b] = s_fill[b];
      p.bin_nspan[lo + b] = s_nsp[b];
    }
  }
  if (lane == 0) p.chunk_nbins[c] = nb;
}

// --------------------------------------------------------------------------
// assignment: LPT and Karmarkar-Karp over a pool held in shared memory
// --------------------------------------------------------------------------

struct LptKey {
  const double* cost;
  const int64_t* id;
  const int32_t* tidx;
  int n;
  __device__ bool operator()(int a, int b) const {
    if (a >= n) return false;
    if (b >= n) return true;
    if (cost[a] != cost[b]) return cost[a] > cost[b];
    if (id[a] != id[b]) return id[a] < id[b];
    return tidx[a] < tidx[b];
  }
};

// Sequential LPT over sorted items by one warp; out[k] = rank of item k.
__device__ void lpt_warp(const int* s_ord, const double* cost, int n, int g, int32_t* out_rank) {
  const int lane = threadIdx.x & 31;
  double load = 0.0;
  for (int q = 0; q < n; ++q) {
    const int k = s_ord[q];
    const double c = cost[k];
    double l = lane < g ? load : __longlong_as_double(0x7ff0000000000000LL);
    int r = lane;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const double l2 = __shfl_xor_sync(MUX_FULL, l, o, 8);
      const int r2 = __shfl_xor_sync(MUX_FULL, r, o, 8);
      if (l2 < l || (l2 == l && r2 < r)) {
        l = l2;
        r = r2;
      }
    }
    r = __shfl_sync(MUX_FULL, r, 0);
    if (lane == r) load = __dadd_rn(load, c);
    if (lane == 0) out_rank[k] = r;
  }
}

// Karmarkar-Karp, g-way largest differencing (pinned reading in
// oracle/planner.py:kk_assign).  One warp; g <= 8; n <= kKkMax.
constexpr int kKkMax = 512;

struct KkSmem {
  double sum[kKkMax * 8];
  int32_t mn[kKkMax * 8];
  int32_t head[kKkMax * 8];
  int32_t tail[kKkMax * 8];
  int32_t next[kKkMax];
  int32_t alive[kKkMax];
  double spread[kKkMax];
  int32_t tmin[kKkMax];
};

__device__ __forceinline__ bool kk_better(double sa, int ma, double sb, int mb) {
  return sa > sb || (sa == sb && ma < mb);
}

__device__ void kk_warp(KkSmem& K, const double* w, int n, int g, int32_t* out_rank) {
  const int lane = threadIdx.x & 31;
  const int INF = INT_MAX;
  for (int t = lane; t < n; t += 32) {
    for (int j = 0; j < g; ++j) {
      K.sum[t * 8 + j] = j == 0 ? w[t] : 0.0;
      K.mn[t * 8 + j] = j == 0 ? t : INF;
      K.head[t * 8 + j] = j == 0 ? t : -1;
      K.tail[t * 8 + j] = j == 0 ? t : -1;
    }
    K.next[t] = -1;
    K.alive[t] = t;
    K.spread[t] = g > 1 ? w[t] : 0.0;
    K.tmin[t] = t;
  }
  __syncwarp();
  int na = n;
  while (na > 1) {
    // top-2 by (spread desc, tmin asc) over the alive list
    int a = -1, b = -1;
    for (int pass = 0; pass < 2; ++pass) {
      double bs = -1.0;
      int bm = INF, bp = -1;
      for (int x = lane; x < na; x += 32) {
        const int t = K.alive[x];
        if (t == a) continue;
        if (bp < 0 || kk_better(K.spread[t], K.tmin[t], bs, bm)) {
          bs = K.spread[t];
          bm = K.tmin[t];
          bp = x;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_xor_sync(MUX_FULL, bs, o);
        const int m2 = __shfl_xor_sync(MUX_FULL, bm, o);
        const int p2 = __shfl_xor_sync(MUX_FULL, bp, o);
        if (p2 >= 0 && (bp < 0 || kk_better(s2, m2, bs, bm))) {
          bs = s2;
          bm = m2;
          bp = p2;
        }
      }
      if (pass == 0) a = K.alive[bp];
      else b = bp;  // position of b in the alive list
    }
    const int tb = K.alive[b];
    // lane j < g owns subset j of A and of B
    double sA = 0, sB = 0;
    int mA = INF, mB = INF, hA = -1, tA = -1, hB = -1, tB = -1;
    if (lane < g) {
      sA = K.sum[a * 8 + lane]; mA = K.mn[a * 8 + lane];
      hA = K.head[a * 8 + lane]; tA = K.tail[a * 8 + lane];
      sB = K.sum[tb * 8 + lane]; mB = K.mn[tb * 8 + lane];
      hB = K.head[tb * 8 + lane]; tB = K.tail[tb * 8 + lane];
    }
    // rank of my A subset in (sum desc, mn asc), of my B subset in (sum asc, mn asc)
    int rA = 0, rB = 0;
    for (int j = 0; j < g; ++j) {
      const double sAj = __shfl_sync(MUX_FULL, sA, j), sBj = __shfl_sync(MUX_FULL, sB, j);
      const int mAj = __shfl_sync(MUX_FULL, mA, j), mBj = __shfl_sync(MUX_FULL, mB, j);
      if (lane < g && j != lane) {
        if (sAj > sA || (sAj == sA && (mAj < mA || (mAj == mA && j < lane)))) ++rA;
        if (sBj < sB || (sBj == sB && (mBj < mB || (mBj == mB && j < lane)))) ++rB;
      }
    }
    __syncwarp();
    // scatter A subsets to slot rA (tuple a), then pair with the B subset of rank rA
    if (lane < g) {
      K.sum[a * 8 + rA] = sA; K.mn[a * 8 + rA] = mA;
      K.head[a * 8 + rA] = hA; K.tail[a * 8 + rA] = tA;
    }
    __syncwarp();
    // stash B subsets by rank in tuple tb's slots (tb is dead after this merge)
    if (lane < g) {
      K.sum[tb * 8 + rB] = sB; K.mn[tb * 8 + rB] = mB;
      K.head[tb * 8 + rB] = hB; K.tail[tb * 8 + rB] = tB;
    }
    __syncwarp();
    if (lane < g) {
      const int j = lane;
      const double s = __dadd_rn(K.sum[a * 8 + j], K.sum[tb * 8 + j]);
      const int m1 = K.mn[a * 8 + j], m2 = K.mn[tb * 8 + j];
      int h1 = K.head[a * 8 + j], t1 = K.tail[a * 8 + j];
      const int h2 = K.head[tb * 8 + j], t2 = K.tail[tb * 8 + j];
      if (h1 < 0) { h1 = h2; t1 = t2; }
      else if (h2 >= 0) { K.next[t1] = h2; t1 = t2; }
      K.sum[a * 8 + j] = s;
      K.mn[a * 8 + j] = m1 < m2 ? m1 : m2;
      K.head[a * 8 + j] = h1;
      K.tail[a * 8 + j] = t1;
    }
    __syncwarp();
    if (lane == 0) {
      double mx = K.sum[a * 8], mi = K.sum[a * 8];
      int tm = K.mn[a * 8];
      for (int j = 1; j < g; ++j) {
        const double s = K.sum[a * 8 + j];
        mx = s > mx ? s : mx;
        mi = s < mi ? s : mi;
        tm = K.mn[a * 8 + j] < tm ? K.mn[a * 8 + j] : tm;
      }
      K.spread[a] = __dsub_rn(mx, mi);
      K.tmin[a] = tm;
      K.alive[b] = K.alive[na - 1];
    }
    --na;
    __syncwarp();
  }
  // final subsets -> ranks by (sum desc, mn asc)
  const int f = K.alive[0];
  double s = 0;
  int m = INF, h = -1;
  if (lane < g) { s = K.sum[f * 8 + lane]; m = K.mn[f * 8 + lane]; h = K.head[f * 8 + lane]; }
  int r = 0;
  for (int j = 0; j < g; ++j) {
    const double sj = __shfl_sync(MUX_FULL, s, j);
    const int mj = __shfl_sync(MUX_FULL, m, j);
    if (lane < g && j != lane && (sj > s || (sj == s && (mj < m || (mj == m && j < lane))))) ++r;
  }
  if (lane < g)
    for (int t = h; t >= 0; t = K.next[t]) out_rank[t] = r;
  __syncwarp();
}

// --------------------------------------------------------------------------
// K_finalize
// --------------------------------------------------------------------------

constexpr int kFinThreads = 1024;

struct LptSmem {
  double cost[4096];
  int64_t id[4096];
  int32_t tidx[4096];
  int32_t ord[4096];
  int32_t rank[4096];
};

__device__ __forceinline__ void set_status(Plan& p, int st) {
  if (threadIdx.x == 0) p.hdr[MUX_H_STATUS] = st;
}

__global__ void __launch_bounds__(kFinThreads) finalize_kernel(mux_plan_cfg cfg,
                                                               const int32_t* lens,
                                                               const int32_t* mods,
                                                               const int64_t* ids,
                                                               const int32_t* carry_seq,
                                                               const int32_t* chunk_off, Plan p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t s_warp[33];
  __shared__ int64_t s_tot[64];
  __shared__ int32_t s_chbase[1025];
  __shared__ int32_t s_nseq;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int S = cfg.S, nc = cfg.n_carry, nch = cfg.n_chunks;

  // ---- A. chunk sequence bases -----------------------------------------
  if (tid == 0) {
    int b = cfg.n_carry_seqs;
    for (int c = 0; c < nch; ++c) {
      s_chbase[c] = b;
      b += p.chunk_nbins[c];
    }
    s_chbase[nch] = b;
    s_nseq = b;
  }
  for (int q = tid; q < cfg.n_carry_seqs; q += nt) p.fills[q] = p.nspans[q] = 0;
  __syncthreads();
  const int n_seq = s_nseq;

  // ---- B. global sequence ids, carry offsets, fills ----------------------
  for (int c = 0; c < nch; ++c) {
    const int lo = chunk_off[c], hi = chunk_off[c + 1];
    const int nb = p.chunk_nbins[c];
    for (int i = lo + tid; i < hi; i += nt) p.seq[i] = s_chbase[c] + p.bin_of[i];
    for (int b = tid; b < nb; b += nt) {
      p.fills[s_chbase[c] + b] = p.bin_fill[lo + b];
      p.nspans[s_chbase[c] + b] = p.bin_nspan[lo + b];
    }
  }
  __syncthreads();
  for (int i = tid; i < nc; i += nt) {
    const int q = carry_seq[i];
    int o = 0, sp = 0;
    for (int j = i - 1; j >= 0 && carry_seq[j] == q; --j) {
      o += lens[j];
      ++sp;
    }
    p.seq[i] = q;
    p.off[i] = o;
    p.span[i] = sp;
    if (i + 1 == nc || carry_seq[i + 1] != q) {
      p.fills[q] = o + lens[i];
      p.nspans[q] = sp + 1;
    }
  }
  __syncthreads();

  // ---- C. errors in the reference's order --------------------------------
  if (tid == 0) p.hdr[MUX_H_N_SEQ] = n_seq;
  const int64_t err_idx = p.hdr[MUX_H_ERR_INDEX];
  if (err_idx >= 0) {
    set_status(p, MUX_ERR_PACKING);
    return;
  }
  if (cfg.mode == MUX_MODE_PACK) {
    set_status(p, MUX_OK);
    return;
  }
  if (cfg.gbs % (cfg.dp * cfg.mbs) != 0 || cfg.dp * cfg.sp != cfg.world) {
    set_status(p, MUX_ERR_CONFIG);
    return;
  }
  if (n_seq < cfg.gbs) {
    set_status(p, MUX_ERR_VALUE);
    return;
  }

  // ---- D. batch geometry ----------------------------------------------------
  const int gbs = cfg.gbs, sp = cfg.sp, W = cfg.world, P = gbs / cfg.dp;
  {
    int64_t carry = 0;
    for (int base = 0; base < gbs; base += nt) {
      const int q = base + tid;
      const int64_t v = q < gbs ? p.fills[q] : 0;
      int64_t tot;
      const int64_t pre = block_excl_scan(v, &tot, s_warp);
      if (q < gbs) p.cu[q] = (int32_t)(carry + pre);
      carry += tot;
    }
    if (tid == 0) p.cu[gbs] = (int32_t)carry;
  }
  for (int x = tid; x < gbs * sp; x += nt) {
    const int q = x / sp, k = x % sp, F = p.fills[q];
    const int base = F / sp, rem = F % sp;
    p.shard_len[x] = base + (k < rem ? 1 : 0);
    p.shard_start[x] = k * base + (k < rem ? k : rem);
  }
  __syncthreads();
  for (int x = tid; x < W; x += nt) {  // x = r*sp + k
    const int r = x / sp, k = x % sp;
    int64_t acc = 0;
    for (int j = 0; j < P; ++j) {
      const int q = r * P + j;
      p.row_base[q * sp + k] = acc;
      acc += p.shard_len[q * sp + k];
    }
    p.llm_rows[x] = acc;
  }
  __syncthreads();

  // ---- E. origin rank / origin_pos --------------------------------------------
  int32_t* s_cnt = reinterpret_cast<int32_t*>(smem);        // [gbs*sp]
  int32_t* s_first = s_cnt + gbs * sp;                       // [gbs*sp]
  for (int x = tid; x < gbs * sp; x += nt) {
    s_cnt[x] = 0;
    s_first[x] = INT_MAX;
  }
  __syncthreads();
  for (int i = tid; i < S; i += nt) {
    const int q = p.seq[i];
    p.group[i] = group_of_mod(mods[i]);
    if (q < gbs) {
      const int F = p.fills[q];
      int pos = p.off[i];
      if (pos > F - 1) pos = F - 1 > 0 ? F - 1 : 0;
      int k = 0;
      for (int kk = 0; kk < sp; ++kk)
        if (p.shard_start[q * sp + kk] <= pos) k = kk;
      p.origin[i] = (q / P) * sp + k;
      p.scratch_a[i] = k;
      if (p.group[i] < 0) {  // text: no encoder rows to move
        p.arena_off[i] = -1;
        p.enc_off[i] = -1;
      }
      atomicAdd(&s_cnt[q * sp + k], 1);
      atomicMin(&s_first[q * sp + k], p.span[i]);
    } else {
      p.origin[i] = -1;
      p.origin_pos[i] = -1;
      p.enc[i] = -1;
      p.arena_off[i] = -1;
      p.enc_off[i] = -1;
      p.llm_rank[i] = -1;
      p.llm_row[i] = -1;
    }
  }
  __syncthreads();
  for (int x = tid; x < W; x += nt) {  // exclusive prefix of counts within (replica, shard)
    const int r = x / sp, k = x % sp;
    int acc = 0;
    for (int j = 0; j < P; ++j) {
      const int q = r * P + j;
      const int c = s_cnt[q * sp + k];
      s_cnt[q * sp + k] = acc;
      acc += c;
    }
  }
  __syncthreads();
  int nbatch = 0;
  for (int i = tid; i < S; i += nt) {
    const int q = p.seq[i];
    if (q < gbs) {
      const int k = p.scratch_a[i];
      p.origin_pos[i] = s_cnt[q * sp + k] + p.span[i] - s_first[q * sp + k];
      ++nbatch;
    }
  }
  {
    int64_t tot;
    block_excl_scan(nbatch, &tot, s_warp);
    if (tid == 0) p.hdr[MUX_H_N_BATCH] = tot;
  }

  // ---- F. loader arena offsets (origin, group) in table order ------------
  auto enc_item = [&](int i) { return p.seq[i] < gbs && p.group[i] >= 0; };
  keyed_scan(
      S, W * MUX_N_GROUPS, [&](int i) { return enc_item(i) ? p.origin[i] * MUX_N_GROUPS + p.group[i] : -1; },
      [&](int i) { return (int64_t)lens[i]; }, [&](int i, int64_t v) { p.arena_off[i] = v; },
      s_tot, s_warp);
  for (int x = tid; x < W * MUX_N_GROUPS; x += nt) p.arena_rows[x] = s_tot[x];
  __syncthreads();

  // ---- G. encoder assignment per pool -------------------------------------------
  LptSmem& ls = *reinterpret_cast<LptSmem*>(smem);
  const int npools = cfg.pooled ? 1 : MUX_N_GROUPS;
  for (int pool = 0; pool < npools; ++pool) {
    auto in_pool = [&](int i) {
      return enc_item(i) && (cfg.pooled || p.group[i] == pool);
    };
    // compact the pool in table order
    keyed_scan(
        S, 1, [&](int i) { return in_pool(i) ? 0 : -1; }, [&](int) { return (int64_t)1; },
        [&](int i, int64_t v) {
          ls.cost[v] = (double)lens[i];
          ls.id[v] = ids[i];
          ls.tidx[v] = i;
        },
        s_tot, s_warp);
    const int m = (int)s_tot[0];
    if (m == 0) continue;
    if (W == 1) {
      for (int k = tid; k < m; k += nt) ls.rank[k] = 0;
    } else if (cfg.method == MUX_LPT) {
      const int mpad = next_pow2(m);
      for (int k = tid; k < mpad; k += nt) ls.ord[k] = k;
      __syncthreads();
      bitonic_sort(ls.ord, mpad, LptKey{ls.cost, ls.id, ls.tidx, m});
      if (tid < 32) lpt_warp(ls.ord, ls.cost, m, W, ls.rank);
    } else {
      if (m > kKkMax) {
        set_status(p, MUX_ERR_VALUE);
        return;
      }
      // KK scratch lives after the LPT arrays (total < 227 KB)
      KkSmem& K = *reinterpret_cast<KkSmem*>(smem + sizeof(LptSmem));
      if (tid < 32) kk_warp(K, ls.cost, m, W, ls.rank);
    }
    __syncthreads();
    for (int k = tid; k < m; k += nt) p.enc[ls.tidx[k]] = ls.rank[k];
    __syncthreads();
  }
  for (int i = tid; i < S; i += nt)
    if (p.seq[i] < gbs && p.group[i] < 0) p.enc[i] = -1;
  __syncthreads();

  // ---- H. encoder order (origin, table index); encoder offsets -----------
  keyed_scan(
      S, W, [&](int i) { return enc_item(i) ? p.origin[i] : -1; }, [&](int) { return (int64_t)1; },
      [&](int i, int64_t v) { p.scratch_b[i] = (int32_t)v; }, s_tot, s_warp);
  if (tid == 0) {
    int64_t acc = 0;
    for (int r = 0; r < W; ++r) {
      const int64_t c = s_tot[r];
      s_tot[32 + r] = acc;
      acc += c;
    }
    s_tot[32 + W] = acc;
  }
  __syncthreads();
  for (int i = tid; i < S; i += nt)
    if (enc_item(i)) p.order[s_tot[32 + p.origin[i]] + p.scratch_b[i]] = i;
  __syncthreads();
  const int n_enc = (int)s_tot[32 + W];
  keyed_scan(
      n_enc, W * MUX_N_GROUPS,
      [&](int t) { const int i = p.order[t]; return p.enc[i] * MUX_N_GROUPS + p.group[i]; },
      [&](int t) { return (int64_t)lens[p.order[t]]; },
      [&](int t, int64_t v) { p.enc_off[p.order[t]] = v; }, s_tot, s_warp);
  for (int x = tid; x < W * MUX_N_GROUPS; x += nt) p.recv_rows[x] = s_tot[x];
  __syncthreads();

  // ---- I. LLM positions, return pieces and segment tables of rank `me` ----
  const int me = cfg.me;
  auto owner_k = [&](int q, int pos) {
    int k = 0;
    for (int kk = 0; kk < sp; ++kk)
      if (p.shard_start[q * sp + kk] <= pos) k = kk;
    return k;
  };
  auto npieces = [&](int i) {
    const int L = lens[i];
    if (L <= 0) return 0;
    const int q = p.seq[i];
    return owner_k(q, p.off[i] + L - 1) - owner_k(q, p.off[i]) + 1;
  };
  for (int i = tid; i < S; i += nt) {
    if (enc_item(i)) {
      const int q = p.seq[i];
      const int pos = p.off[i];
      const int k = owner_k(q, pos < p.fills[q] ? pos : (p.fills[q] > 0 ? p.fills[q] - 1 : 0));
      p.llm_rank[i] = (q / P) * sp + k;
      p.llm_row[i] = p.row_base[q * sp + k] + pos - p.shard_start[q * sp + k];
    } else if (p.seq[i] < gbs) {
      p.llm_rank[i] = -1;
      p.llm_row[i] = -1;
    }
  }
  // dispatch segments: samples of `me` with rows to move, table order
  keyed_scan(
      S, 1, [&](int i) { return enc_item(i) && p.origin[i] == me && lens[i] > 0 ? 0 : -1; },
      [&](int) { return (int64_t)1; },
      [&](int i, int64_t v) {
        p.dsrc[v] = p.arena_off[i];
        p.ddst[v] = p.enc_off[i];
        p.drows[v] = lens[i];
        p.dgroup[v] = p.group[i];
        p.drank[v] = p.enc[i];
      },
      s_tot, s_warp);
  const int nd = (int)s_tot[0];
  // return pieces: samples encoded on `me`, split at Ulysses shard borders
  keyed_scan(
      S, 1, [&](int i) { return enc_item(i) && p.enc[i] == me ? 0 : -1; },
      [&](int i) { return (int64_t)npieces(i); },
      [&](int i, int64_t v) {
        const int q = p.seq[i], L = lens[i];
        int t = 0, slot = (int)v;
        while (t < L) {
          const int pos = p.off[i] + t;
          const int k = owner_k(q, pos);
          const int end = p.shard_start[q * sp + k] + p.shard_len[q * sp + k];
          const int n = (L - t) < (end - pos) ? (L - t) : (end - pos);
          p.rsrc[slot] = p.enc_off[i] + t;
          p.rdst[slot] = p.row_base[q * sp + k] + pos - p.shard_start[q * sp + k];
          p.rrows[slot] = n;
          p.rgroup[slot] = p.group[i];
          p.rrank[slot] = (q / P) * sp + k;
          ++slot;
          t += n;
        }
      },
      s_tot, s_warp);
  const int nr = (int)s_tot[0];

  // chunk prefix + chunk maps for both tables
  const int64_t CH = cfg.chunk_bytes > 0 ? cfg.chunk_bytes : kDefaultChunkBytes;
  for (int which = 0; which < 2; ++which) {
    const int n = which == 0 ? nd : nr;
    int64_t* rows = which == 0 ? p.drows : p.rrows;
    int32_t* grp = which == 0 ? p.dgroup : p.rgroup;
    int32_t* rk = which == 0 ? p.drank : p.rrank;
    int64_t* c0 = which == 0 ? p.dchunk0 : p.rchunk0;
    int32_t* cmap = which == 0 ? p.dchunk_seg : p.rchunk_seg;
    const int32_t* rb = which == 0 ? cfg.row_bytes_in : cfg.row_bytes_ret;
    int64_t carry = 0, bytes = 0, remote = 0;
    for (int base = 0; base < n; base += nt) {
      const int s = base + tid;
      int64_t nbytes = 0, nchk = 0;
      if (s < n) {
        nbytes = rows[s] * (int64_t)rb[grp[s]];
        nchk = (nbytes + CH - 1) / CH;
      }
      int64_t tot;
      const int64_t pre = block_excl_scan(nchk, &tot, s_warp);
      if (s < n) c0[s] = carry + pre;
      carry += tot;
      int64_t tb, trm;
      block_excl_scan(nbytes, &tb, s_warp);
      block_excl_scan(s < n && rk[s] != me ? nbytes : 0, &trm, s_warp);
      bytes += tb;
      remote += trm;
    }
    if (tid == 0) {
      c0[n] = carry;
      p.hdr[which == 0 ? MUX_H_DISPATCH_CHUNKS : MUX_H_RETURN_CHUNKS] = carry;
      p.hdr[which == 0 ? MUX_H_DISPATCH_BYTES : MUX_H_RETURN_BYTES] = bytes;
      p.hdr[which == 0 ? MUX_H_DISPATCH_REMOTE : MUX_H_RETURN_REMOTE] = remote;
    }
    __syncthreads();
    if (carry > cfg.max_chunks) {
      set_status(p, MUX_ERR_RUNTIME);
      return;
    }
    const int warp = tid >> 5, lane = tid & 31;
    for (int s = warp; s < n; s += nt / 32)
      for (int64_t c = c0[s] + lane; c < c0[s + 1]; c += 32) cmap[c] = s;
  }
  if (tid == 0) {
    p.hdr[MUX_H_N_DISPATCH] = nd;
    p.hdr[MUX_H_N_RETURN] = nr;
    p.hdr[MUX_H_RECV_ROWS0] = p.recv_rows[me * MUX_N_GROUPS + 0];
    p.hdr[MUX_H_RECV_ROWS1] = p.recv_rows[me * MUX_N_GROUPS + 1];
    p.hdr[MUX_H_STATUS] = MUX_OK;
  }
}

// Stand-alone partition (kk_partition / LPT) of one pool.
__global__ void __launch_bounds__(kFinThreads) assign_kernel(int method, const double* w,
                                                             const int64_t* ids, int n, int g,
                                                             int32_t* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  LptSmem& ls = *reinterpret_cast<LptSmem*>(smem);
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    ls.cost[k] = w[k];
    ls.id[k] = ids ? ids[k] : k;
    ls.tidx[k] = k;
  }
  __syncthreads();
  if (g == 1) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) ls.rank[k] = 0;
  } else if (method == MUX_LPT) {
    const int npad = next_pow2(n > 0 ? n : 1);
    for (int k = threadIdx.x; k < npad; k += blockDim.x) ls.ord[k] = k;
    __syncthreads();
    bitonic_sort(ls.ord, npad, LptKey{ls.cost, ls.id, ls.tidx, n});
    if (threadIdx.x < 32) lpt_warp(ls.ord, ls.cost, n, g, ls.rank);
  } else {
    KkSmem& K = *reinterpret_cast<KkSmem*>(smem + sizeof(LptSmem));
    if (threadIdx.x < 32) kk_warp(K, ls.cost, n, g, ls.rank);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) out[k] = ls.rank[k];
}

static size_t finalize_smem() {
  return sizeof(LptSmem) + sizeof(KkSmem);  // 206,848 B < 227 KB
}

}  // namespace mux

using namespace mux;

extern "C" int mux_plan_layout_of(const mux_plan_cfg* cfg, mux_plan_layout* out) {
  if (!cfg || !out) {
    set_error("null argument");
    return MUX_ERR_VALUE;
  }
  return compute_layout(*cfg, out);
}

extern "C" int mux_plan_step(const mux_plan_cfg* cfg, const int32_t* lens, const int32_t* mods,
                             const int64_t* ids, const int32_t* carry_seq,
                             const int32_t* chunk_off, void* plan, size_t plan_bytes,
                             void* stream) {
  mux_plan_layout L;
  int st = compute_layout(*cfg, &L);
  if (st) return st;
  if ((int64_t)plan_bytes < L.total) {
    set_error("plan buffer of %zu bytes, need %lld", plan_bytes, (long long)L.total);
    return MUX_ERR_VALUE;
  }
  if (cfg->n_chunks > 1024) {
    set_error("more than 1024 chunks in one step");
    return MUX_ERR_VALUE;
  }
  if (cfg->mode == MUX_MODE_STEP && (cfg->me < 0 || cfg->me >= cfg->world)) {
    set_error("rank %d outside world %d", cfg->me, cfg->world);
    return MUX_ERR_VALUE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Plan p = make_plan(plan, L);
  MUX_CUDA(cudaMemsetAsync(p.hdr, 0xff, 8 * MUX_H_SLOTS, s));
  static bool attr_done = false;
  if (!attr_done) {
    MUX_CUDA(cudaFuncSetAttribute(ffd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  4096 * 24));
    MUX_CUDA(cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)finalize_smem()));
    MUX_CUDA(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)finalize_smem()));
    attr_done = true;
  }
  if (cfg->n_chunks > 0) {
    // worst chunk size bounds the shared memory: npad * (8 + 4*4)
    int maxn = cfg->S - cfg->n_carry;
    int npad = 1;
    while (npad < maxn) npad <<= 1;
    ffd_kernel<<<cfg->n_chunks, kFfdThreads, (size_t)npad * 24, s>>>(*cfg, lens, ids, chunk_off,
                                                                      p);
    MUX_CUDA(cudaGetLastError());
  }
  finalize_kernel<<<1, kFinThreads, finalize_smem(), s>>>(*cfg, lens, mods, ids, carry_seq,
                                                           chunk_off, p);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

extern "C" int mux_plan_check(const mux_plan_cfg* cfg, const int64_t* h, const int64_t* ids,
                              const int32_t* lens) {
  const int64_t st = h[MUX_H_STATUS];
  if (st == MUX_OK) return MUX_OK;
  switch (st) {
    case MUX_ERR_PACKING: {
      const int64_t i = h[MUX_H_ERR_INDEX];
      set_error("sample %lld (%d tokens) exceeds capacity %d", (long long)ids[i], lens[i],
                cfg->capacity);
      return MUX_ERR_PACKING;
    }
    case MUX_ERR_CONFIG:
      if (cfg->dp * cfg->sp != cfg->world && cfg->gbs % (cfg->dp * cfg->mbs) == 0)
        set_error("llm dp %d x sp %d != world %d", cfg->dp, cfg->sp, cfg->world);
      else
        set_error("global batch %d not divisible by dp %d x microbatch size %d", cfg->gbs,
                  cfg->dp, cfg->mbs);
      return MUX_ERR_CONFIG;
    case MUX_ERR_VALUE:
      if (h[MUX_H_N_SEQ] < cfg->gbs) {
        set_error("need %d sequences, have %lld", cfg->gbs, (long long)h[MUX_H_N_SEQ]);
      } else {
        set_error("encoder pool larger than the KK limit %d", kKkMax);
      }
      return MUX_ERR_VALUE;
    case MUX_ERR_RUNTIME:
      set_error("copy chunk map overflow (max_chunks %d)", cfg->max_chunks);
      return MUX_ERR_RUNTIME;
    default:
      set_error("plan did not complete (status %lld)", (long long)st);
      return MUX_ERR_RUNTIME;
  }
}

extern "C" size_t mux_assign_scratch_bytes(int32_t, int32_t) { return 0; }

extern "C" int mux_assign(int32_t method, const double* w, const int64_t* ids, int32_t n,
                          int32_t g, int32_t* out, void*, void* stream) {
  if (g < 1 || g > 8) {
    set_error("group count %d outside 1..8", g);
    return MUX_ERR_VALUE;
  }
  if (n < 0 || n > 4096 || (method == MUX_KK && n > kKkMax)) {
    set_error("%d weights exceed the device limit", n);
    return MUX_ERR_VALUE;
  }
  if (n == 0) return MUX_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MUX_CUDA(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)finalize_smem()));
  assign_kernel<<<1, kFinThreads, finalize_smem(), s>>>(method, w, ids, n, g, out);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
