// Device planner for one step of the encoder<->LLM data path (sm_100a).
//
// One launch, `plan_kernel`, grid = one CTA per drawn chunk:
//  part 1  every CTA packs its chunk: bitonic sort by (-len, id, index) in
//          shared memory, then a warp-synchronous first fit with the bins in
//          registers (reference: pkg/src/muxsim/workload.py:240-262);
//  part 2  the last CTA to finish (atomic ticket) finalises the whole step:
//          carry spans, global sequence ids, errors in the reference's order
//          (workload.py:245-248, :269-275), batch slice and replica owner
//          (:265-280, :177-180), Ulysses shard geometry,
//          origins, loader-arena offsets, encoder assignment per pool (LPT or
//          KK), encoder order, return pieces and the
//          segment tables of rank `me` that drive the copy kernels.
// For steps of up to kSmallS samples every per-sample array of part 2 lives
// in shared memory (written back once at the end); larger steps work on the
// plan blob in global memory.  Integer / exact-double arithmetic only, so
// every rank computes the identical plan and pushes rows without exchanging
// counts.

#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "mux_common.cuh"

namespace mux {

constexpr int kSmallS = 1024;   // per-sample state in shared memory up to this S
constexpr int kThreads = 1024;
constexpr int kRegSlots = 8;    // first-fit bins in registers: 32 lanes x 8 = 256
constexpr int kKkMax = 512;     // KK pool limit (one warp, tuples in shared memory)
constexpr int kMaxChunks = 1024;

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
  if (c.n_chunks > kMaxChunks) {
    set_error("more than %d chunks in one step", kMaxChunks);
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
    if (c.ret_mode == MUX_RET_STAGED && c.sp != 1) {
      set_error("staged projector return needs Ulysses sp == 1 (got %d)", c.sp);
      return MUX_ERR_VALUE;
    }
    if (c.lssp_sp < 0 || c.lssp_sp > MUX_LSSP_MAX ||
        (c.lssp_sp > 0 && (c.world % c.lssp_sp || c.ret_mode != MUX_RET_FINAL || c.lssp_eta < 0))) {
      set_error("LSSP group %d: need 1..%d dividing world %d, eta >= 0, final-row return",
                c.lssp_sp, MUX_LSSP_MAX, c.world);
      return MUX_ERR_VALUE;
    }
    const int rg = c.reorder_group > 0 ? c.reorder_group : c.world;
    if (c.reorder_group < 0 || c.world % rg || (c.lssp_sp > 0 && rg % c.lssp_sp)) {
      set_error("reorder group %d: need 0 (world) or a divisor of world %d that LSSP groups "
                "(%d) divide", c.reorder_group, c.world, c.lssp_sp);
      return MUX_ERR_VALUE;
    }
    if (c.cost_model != MUX_COST_TOKENS &&
        (c.cost_model != MUX_COST_FLOPS || !(c.cost_lin[0] >= 0) || !(c.cost_lin[1] >= 0) ||
         !(c.cost_quad[0] >= 0) || !(c.cost_quad[1] >= 0))) {
      set_error("cost model %d: need tokens (0) or flops (1) with non-negative parameters",
                c.cost_model);
      return MUX_ERR_VALUE;
    }
    if (c.reshard != MUX_RESHARD_ULYSSES &&
        (c.reshard != MUX_RESHARD_CP_HYBRID || c.ret_mode != MUX_RET_FINAL ||
         c.cp_threshold < 0 || c.sp > 8)) {
      set_error("reshard %d: need Ulysses (0) or CpHybrid (1) with final-row return, "
                "cp_threshold >= 0, sp <= 8", c.reshard);
      return MUX_ERR_VALUE;
    }
  } else if (c.lssp_sp != 0 || c.reshard != MUX_RESHARD_ULYSSES || c.text_embed) {
    set_error("LSSP, CpHybrid and text rows apply to step plans only");
    return MUX_ERR_VALUE;
  }
  const int64_t S = c.S > 0 ? c.S : 1;
  const int64_t nch = c.n_chunks > 0 ? c.n_chunks : 1;
  const int64_t mseq = max_seq_of(c);
  const int64_t gb = (c.gbs > 0 ? c.gbs : 1) * (c.sp > 0 ? c.sp : 1);
  const int64_t W = (c.world > 0 ? c.world : 1);
  const int64_t R = max_ret_of(c);
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    int64_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L->header = take(8 * MUX_H_SLOTS);
  L->sync = take(8);
  L->seq = take(4 * S);
  L->off = take(4 * S);
  L->span = take(4 * S);
  L->origin = take(4 * S);
  L->origin_pos = take(4 * S);
  L->group = take(4 * S);
  L->enc = take(4 * S);
  L->arena_off = take(8 * S);
  L->enc_off = take(8 * S);
  L->stage_off = take(8 * S);
  L->llm_rank = take(4 * S);
  L->llm_row = take(8 * S);
  L->bin_fill = take(4 * S);
  L->bin_nspan = take(4 * S);
  L->bin_of = take(4 * S);
  L->chunk_nbins = take(4 * nch);
  L->chunk_err = take(4 * nch);
  L->fills = take(4 * mseq);
  L->nspans = take(4 * mseq);
  L->cu = take(4 * (gb + 1));
  L->shard_len = take(4 * gb);
  L->shard_start = take(4 * gb);
  L->row_base = take(8 * gb);
  L->arena_rows = take(8 * W * MUX_N_GROUPS);
  L->recv_rows = take(8 * W * MUX_N_GROUPS);
  L->stage_rows = take(8 * W * MUX_N_GROUPS);
  L->llm_rows = take(8 * W);
  L->order = take(4 * S);
  L->scratch_a = take(4 * S);
  L->scratch_b = take(4 * S);
  const int64_t D = c.S > 0 ? max_disp_of(c) : 1;
  L->dseg_src_row = take(8 * D);
  L->dseg_dst_row = take(8 * D);
  L->dseg_rows = take(8 * D);
  L->dseg_group = take(4 * D);
  L->dseg_dst_rank = take(4 * D);
  L->dseg_chunk0 = take(8 * (D + 1));
  L->rseg_src_row = take(8 * R);
  L->rseg_dst_row = take(8 * R);
  L->rseg_rows = take(8 * R);
  L->rseg_group = take(4 * R);
  L->rseg_dst_rank = take(4 * R);
  L->rseg_chunk0 = take(8 * (R + 1));
  L->gseg_src_row = take(8 * R);
  L->gseg_dst_row = take(8 * R);
  L->gseg_rows = take(8 * R);
  L->gseg_group = take(4 * R);
  L->gseg_dst_rank = take(4 * R);
  L->gseg_chunk0 = take(8 * (R + 1));
  L->lssp_state = take(4 * S);
  L->lssp_row = take(8 * S * MUX_LSSP_MAX);
  const int64_t SP = S * (c.sp > 0 ? c.sp : 1);
  L->lp_n = take(4 * S);
  L->lp_k = take(4 * SP);
  L->lp_t0 = take(4 * SP);
  L->lp_len = take(4 * SP);
  L->lp_row = take(8 * SP);
  const int64_t RT = S * ((c.sp > 0 ? c.sp : 1) + 1);
  L->text_off = take(8 * S);
  L->tseg_src = take(8 * RT);
  L->tseg_dst = take(8 * RT);
  L->tseg_rows = take(8 * RT);
  L->tseg_row0 = take(8 * (RT + 1));
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
  p.ticket = at<uint32_t>(b, L.sync);
  p.seq = at<int32_t>(b, L.seq);
  p.off = at<int32_t>(b, L.off);
  p.span = at<int32_t>(b, L.span);
  p.origin = at<int32_t>(b, L.origin);
  p.origin_pos = at<int32_t>(b, L.origin_pos);
  p.group = at<int32_t>(b, L.group);
  p.enc = at<int32_t>(b, L.enc);
  p.arena_off = at<int64_t>(b, L.arena_off);
  p.enc_off = at<int64_t>(b, L.enc_off);
  p.stage_off = at<int64_t>(b, L.stage_off);
  p.llm_rank = at<int32_t>(b, L.llm_rank);
  p.llm_row = at<int64_t>(b, L.llm_row);
  p.bin_fill = at<int32_t>(b, L.bin_fill);
  p.bin_nspan = at<int32_t>(b, L.bin_nspan);
  p.bin_of = at<int32_t>(b, L.bin_of);
  p.chunk_nbins = at<int32_t>(b, L.chunk_nbins);
  p.chunk_err = at<int32_t>(b, L.chunk_err);
  p.fills = at<int32_t>(b, L.fills);
  p.nspans = at<int32_t>(b, L.nspans);
  p.cu = at<int32_t>(b, L.cu);
  p.shard_len = at<int32_t>(b, L.shard_len);
  p.shard_start = at<int32_t>(b, L.shard_start);
  p.row_base = at<int64_t>(b, L.row_base);
  p.arena_rows = at<int64_t>(b, L.arena_rows);
  p.recv_rows = at<int64_t>(b, L.recv_rows);
  p.stage_rows = at<int64_t>(b, L.stage_rows);
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
  p.rsrc = at<int64_t>(b, L.rseg_src_row);
  p.rdst = at<int64_t>(b, L.rseg_dst_row);
  p.rrows = at<int64_t>(b, L.rseg_rows);
  p.rgroup = at<int32_t>(b, L.rseg_group);
  p.rrank = at<int32_t>(b, L.rseg_dst_rank);
  p.rchunk0 = at<int64_t>(b, L.rseg_chunk0);
  p.gsrc = at<int64_t>(b, L.gseg_src_row);
  p.gdst = at<int64_t>(b, L.gseg_dst_row);
  p.grows = at<int64_t>(b, L.gseg_rows);
  p.ggroup = at<int32_t>(b, L.gseg_group);
  p.grank = at<int32_t>(b, L.gseg_dst_rank);
  p.gchunk0 = at<int64_t>(b, L.gseg_chunk0);
  p.lssp_state = at<int32_t>(b, L.lssp_state);
  p.lssp_row = at<int64_t>(b, L.lssp_row);
  p.lp_n = at<int32_t>(b, L.lp_n);
  p.lp_k = at<int32_t>(b, L.lp_k);
  p.lp_t0 = at<int32_t>(b, L.lp_t0);
  p.lp_len = at<int32_t>(b, L.lp_len);
  p.lp_row = at<int64_t>(b, L.lp_row);
  p.text_off = at<int64_t>(b, L.text_off);
  p.tsrc = at<int64_t>(b, L.tseg_src);
  p.tdst = at<int64_t>(b, L.tseg_dst);
  p.trows = at<int64_t>(b, L.tseg_rows);
  p.trow0 = at<int64_t>(b, L.tseg_row0);
  return p;
}

Plan make_plan_const(const void* b, const mux_plan_layout& L) {
  return make_plan(const_cast<void*>(b), L);
}

// Phase timestamps (globaltimer, ns): stamp slot 16..25 -> header slot 20..29.
__device__ __forceinline__ void stamp(Plan& p, int slot) {
  if (threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.hdr[MUX_H_STAMP0 + slot - 16] = (int64_t)t;
  }
}

// --------------------------------------------------------------------------
// sort keys, LPT and Karmarkar-Karp
// --------------------------------------------------------------------------

struct FfdKey {  // (-len, id, index) ascending; padding (>= n) last
  const int32_t* len;
  const int64_t* id;
  int n;
  __device__ bool operator()(int a, int b) const {
    if (a >= n) return false;
    if (b >= n) return true;
    if (len[a] != len[b]) return len[a] > len[b];
    if (id[a] != id[b]) return id[a] < id[b];
    return a < b;
  }
};

struct PoolKey {  // (pool, -cost, id, table index) ascending; padding last
  const int32_t* pool;
  const double* cost;
  const int64_t* id;
  const int32_t* tidx;
  int n;
  __device__ bool operator()(int a, int b) const {
    if (a >= n) return false;
    if (b >= n) return true;
    if (pool[a] != pool[b]) return pool[a] < pool[b];
    if (cost[a] != cost[b]) return cost[a] > cost[b];
    if (id[a] != id[b]) return id[a] < id[b];
    return tidx[a] < tidx[b];
  }
};

// Sequential LPT over sorted items by one warp; out[k] = rank of item k.
__device__ void lpt_warp(const int* s_ord, const double* cost, int n, int g, int32_t* out_rank,
                         const double* init = nullptr) {
  const int lane = threadIdx.x & 31;
  double load = init != nullptr && lane < g ? init[lane] : 0.0;
  int nxt = n > 0 ? s_ord[0] : 0;
  double nc = n > 0 ? cost[nxt] : 0.0;
  for (int q = 0; q < n; ++q) {
    const int k = nxt;
    const double c = nc;
    if (q + 1 < n) {
      nxt = s_ord[q + 1];
      nc = cost[nxt];
    }
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

// Locality-first LPT over sorted items by one warp: pass 1 keeps each item on
// its origin rank while that rank's kept load stays within the balanced load
// T = sum / g; pass 2 places the rest by LPT on top of the kept loads.  With
// integer-valued costs every sum is exact, so it matches the CPU oracle bit
// for bit (oracle/planner.py:lpt_local_assign).
__device__ void lpt_local_warp(const int* s_ord, const double* cost, const int32_t* origin, int n,
                               int g, int32_t* out_rank, int32_t* s_kept_flag, bool remote_w) {
  const int lane = threadIdx.x & 31;
  double part = 0.0;
  for (int q = lane; q < n; q += 32) part += cost[s_ord[q]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(MUX_FULL, part, o);
  const double T = __ddiv_rn(part, (double)g);
  double kept = 0.0;  // lane k < g: kept load of rank k
  for (int q = 0; q < n; ++q) {
    const int k = s_ord[q];
    const double c = cost[k];
    const int o = origin[k];
    const double ko = __shfl_sync(MUX_FULL, kept, o);
    const bool keep = __dadd_rn(ko, c) <= T;
    if (keep && lane == o) kept = __dadd_rn(kept, c);
    if (lane == 0) {
      s_kept_flag[q] = keep;
      if (keep) out_rank[k] = o;
    }
  }
  __syncwarp();
  double load = kept;
  for (int q = 0; q < n; ++q) {
    if (s_kept_flag[q]) continue;
    const int k = s_ord[q];
    const double c = cost[k];
    // remote_w: the item costs 9/8 c on a rank other than its origin; the rank
    // with the smallest resulting load wins (lowest rank on ties).  Costs are
    // integers, so every value is a multiple of 1/8 and exact.
    const double ce = remote_w && lane != origin[k] ? __dmul_rn(c, 1.125) : c;
    double l = lane < g ? __dadd_rn(load, ce) : __longlong_as_double(0x7ff0000000000000LL);
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
    if (lane == r) load = __dadd_rn(load, ce);
    if (lane == 0) out_rank[k] = r;
  }
  __syncwarp();
}

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

// Karmarkar-Karp, g-way largest differencing (pinned reading in
// oracle/planner.py:kk_assign).  One warp; g <= 8; n <= kKkMax.
// w[t] / out_rank[t] for t < n.
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
    int a = -1, b = -1;  // top-2 by (spread desc, tmin asc) over the alive list
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
    double sA = 0, sB = 0;  // lane j < g owns subset j of A and of B
    int mA = INF, mB = INF, hA = -1, tA = -1, hB = -1, tB = -1;
    if (lane < g) {
      sA = K.sum[a * 8 + lane]; mA = K.mn[a * 8 + lane];
      hA = K.head[a * 8 + lane]; tA = K.tail[a * 8 + lane];
      sB = K.sum[tb * 8 + lane]; mB = K.mn[tb * 8 + lane];
      hB = K.head[tb * 8 + lane]; tB = K.tail[tb * 8 + lane];
    }
    // rank of my A subset in (sum desc, mn asc), of my B subset in (sum asc, mn asc);
    // identical (empty) subsets tie-break by lane
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
    if (lane < g) {  // A subsets to slot rA of tuple a, B subsets to slot rB of tuple tb
      K.sum[a * 8 + rA] = sA; K.mn[a * 8 + rA] = mA;
      K.head[a * 8 + rA] = hA; K.tail[a * 8 + rA] = tA;
      K.sum[tb * 8 + rB] = sB; K.mn[tb * 8 + rB] = mB;
      K.head[tb * 8 + rB] = hB; K.tail[tb * 8 + rB] = tB;
    }
    __syncwarp();
    if (lane < g) {  // pair A's j-th largest with B's j-th smallest
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
  const int f = K.alive[0];  // final subsets -> ranks by (sum desc, mn asc)
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
// block-wide multi-key scan: one element per thread per call, K <= 16 keys.
// Returns the exclusive prefix of `val` among earlier elements (this call
// and previous calls) with the same key; s_carry[k] accumulates per-key
// totals across calls (caller zeroes it).  Three barriers per call.
// --------------------------------------------------------------------------
constexpr int kMaxKeys = 16;

__device__ __forceinline__ int64_t multi_scan(int key, int64_t val, int K, int64_t* s_wk,
                                              int64_t* s_carry) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t mine_incl = 0;
#pragma unroll
  for (int k = 0; k < kMaxKeys; ++k) {
    if (k >= K) break;
    int64_t x = key == k ? val : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(MUX_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wk[w * kMaxKeys + k] = x;
    if (key == k) mine_incl = x;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    int64_t run = s_carry[k];
    for (int j = 0; j < nw; ++j) {
      const int64_t t = s_wk[j * kMaxKeys + k];
      s_wk[j * kMaxKeys + k] = run;
      run += t;
    }
    s_carry[k] = run;
  }
  __syncthreads();
  const int64_t r = (key >= 0 && key < K) ? s_wk[w * kMaxKeys + key] + mine_incl - val : 0;
  __syncthreads();
  return r;
}

// --------------------------------------------------------------------------
// part 1: first-fit decreasing of one chunk (whole CTA sorts; warp 0 places)
// --------------------------------------------------------------------------

__device__ void ffd_chunk(const mux_plan_cfg& cfg, const int32_t* lens, const int64_t* ids,
                          const int32_t* chunk_off, Plan& p, unsigned char* smem,
                          int64_t* s_warp) {
  __shared__ int s_err;
  const int c = blockIdx.x;
  const int lo = chunk_off[c], n = chunk_off[c + 1] - lo;
  const int npad = next_pow2(n > 0 ? n : 1);
  int64_t* s_id = reinterpret_cast<int64_t*>(smem);
  int32_t* s_len = reinterpret_cast<int32_t*>(s_id + npad);
  int32_t* s_ord = s_len + npad;
  int32_t* s_fill = s_ord + npad;  // shared-memory first fit (many bins) only
  int32_t* s_nsp = s_fill + npad;
  const int cap = cfg.capacity;
  if (threadIdx.x == 0) s_err = INT_MAX;
  __syncthreads();
  int64_t my_total = 0;
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    if (i < n) {
      const int L = lens[lo + i];
      s_len[i] = L;
      s_id[i] = ids[lo + i];
      my_total += L;
      if (L > cap) atomicMin(&s_err, lo + i);  // first offender in table order
    }
    s_ord[i] = i;
  }
  int64_t total;
  block_excl_scan(my_total, &total, s_warp);  // (its barriers also publish the loads)
  bitonic_sort(s_ord, npad, FfdKey{s_len, s_id, n});
  if (threadIdx.x == 0) p.chunk_err[c] = s_err;

  // first fit never leaves two bins at most half full: #bins <= 2*total/cap + 1
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
// part 2: finalise (one CTA)
// --------------------------------------------------------------------------

struct Work {  // per-sample working arrays: shared memory (S <= kSmallS) or the plan blob
  int32_t *len, *seq, *off, *span, *grp, *org, *k, *opos, *enc, *within, *order;
  int64_t *id, *aoff, *eoff;
  int32_t *fills, *nspans;
};

struct SmemPlan {  // byte offsets of the finalize-phase shared-memory regions
  int work, shard, lpt, kk, total;
};

__host__ __device__ inline SmemPlan smem_plan(int S, int n_seq_max, int gb, int method) {
  SmemPlan L;
  int o = 0;
  L.work = o;
  if (S <= kSmallS) o += 68 * S + 8 * n_seq_max;
  o = (int)align_up(o, 16);
  L.shard = o;  // shard start / length per (sequence, shard), phases D..I
  o += 8 * gb;
  o = (int)align_up(o, 16);
  L.lpt = o;  // phase E counters, then the pool sort (phase G)
  int spad = 1;
  while (spad < S) spad <<= 1;
  o += 40 * spad > 8 * gb ? 40 * spad : 8 * gb;  // cost, id, tidx, pool, ord, rank, org, flag
  o = (int)align_up(o, 16);
  L.kk = o;
  if (method == MUX_KK) o += (int)sizeof(KkSmem);
  L.total = o;
  return L;
}

__device__ __forceinline__ void set_status(Plan& p, int st) {
  if (threadIdx.x == 0) p.hdr[MUX_H_STATUS] = st;
}

// write the shared-memory working arrays back to the plan blob
__device__ void emit(const mux_plan_cfg& cfg, Plan& p, const Work& w, bool small, int n_seq,
                     bool full) {
  if (!small) return;
  for (int i = threadIdx.x; i < cfg.S; i += blockDim.x) {
    p.seq[i] = w.seq[i];
    p.off[i] = w.off[i];
    p.span[i] = w.span[i];
    if (full) {
      p.group[i] = w.grp[i];
      p.origin[i] = w.org[i];
      p.origin_pos[i] = w.opos[i];
      p.enc[i] = w.enc[i];
      p.arena_off[i] = w.aoff[i];
      p.enc_off[i] = w.eoff[i];
    }
  }
  for (int q = threadIdx.x; q < n_seq; q += blockDim.x) {
    p.fills[q] = w.fills[q];
    p.nspans[q] = w.nspans[q];
  }
}

__device__ void finalize(const mux_plan_cfg& cfg, const int32_t* lens, const int32_t* mods,
                         const int64_t* ids, const int32_t* carry_seq, const int32_t* chunk_off,
                         Plan& p, unsigned char* smem, int64_t* s_warp) {
  __shared__ int64_t s_wk[32 * kMaxKeys];
  __shared__ int64_t s_carry[kMaxKeys];
  __shared__ int32_t s_chbase[kMaxChunks + 1];
  __shared__ int32_t s_misc[8 + kMaxKeys + 1];  // scalars, then the pool offsets of G
  const int tid = threadIdx.x, nt = blockDim.x;
  const int S = cfg.S, nc = cfg.n_carry, nch = cfg.n_chunks, W = cfg.world;
  const int max_seq = cfg.n_carry_seqs + (S - nc) + 1;
  const bool small = S <= kSmallS;
  const SmemPlan SL = smem_plan(S, max_seq, cfg.gbs * cfg.sp, cfg.method);
  stamp(p, 17);

  // ---- working storage -----------------------------------------------------
  Work w;
  if (small) {
    unsigned char* b = smem + SL.work;
    w.id = reinterpret_cast<int64_t*>(b);
    w.aoff = w.id + S;
    w.eoff = w.aoff + S;
    int32_t* q = reinterpret_cast<int32_t*>(w.eoff + S);
    w.len = q; q += S;
    w.seq = q; q += S;
    w.off = q; q += S;
    w.span = q; q += S;
    w.grp = q; q += S;
    w.org = q; q += S;
    w.k = q; q += S;
    w.opos = q; q += S;
    w.enc = q; q += S;
    w.within = q; q += S;
    w.order = q; q += S;
    w.fills = q; q += max_seq;
    w.nspans = q;
    for (int i = tid; i < S; i += nt) {
      w.len[i] = lens[i];
      w.id[i] = ids[i];
    }
  } else {
    w.len = const_cast<int32_t*>(lens);
    w.id = const_cast<int64_t*>(ids);
    w.seq = p.seq; w.off = p.off; w.span = p.span; w.grp = p.group; w.org = p.origin;
    w.k = p.scratch_a; w.opos = p.origin_pos; w.enc = p.enc; w.within = p.scratch_b;
    w.order = p.order; w.aoff = p.arena_off; w.eoff = p.enc_off;
    w.fills = p.fills; w.nspans = p.nspans;
  }

  // ---- A. chunk sequence bases, first oversize sample ------------------------
  if (tid == 0) {
    int b = cfg.n_carry_seqs, err = INT_MAX;
    for (int c = 0; c < nch; ++c) {
      s_chbase[c] = b;
      b += __ldcg(p.chunk_nbins + c);
      const int e = __ldcg(p.chunk_err + c);
      err = e < err ? e : err;
    }
    s_chbase[nch] = b;
    s_misc[0] = b;    // n_seq
    s_misc[1] = err;  // first oversize table index
  }
  for (int q = tid; q < cfg.n_carry_seqs; q += nt) w.fills[q] = w.nspans[q] = 0;
  __syncthreads();
  const int n_seq = s_misc[0];

  // ---- B. global sequence ids, carry spans, fills -----------------------------
  for (int c = 0; c < nch; ++c) {
    const int lo = chunk_off[c], hi = chunk_off[c + 1];
    const int base = s_chbase[c], nb = s_chbase[c + 1] - base;
    for (int i = lo + tid; i < hi; i += nt) {
      w.seq[i] = base + __ldcg(p.bin_of + i);
      w.off[i] = __ldcg(p.off + i);
      w.span[i] = __ldcg(p.span + i);
    }
    for (int b = tid; b < nb; b += nt) {
      w.fills[base + b] = __ldcg(p.bin_fill + lo + b);
      w.nspans[base + b] = __ldcg(p.bin_nspan + lo + b);
    }
  }
  __syncthreads();
  for (int i = tid; i < nc; i += nt) {
    const int q = carry_seq[i];
    int o = 0, sp = 0;
    for (int j = i - 1; j >= 0 && carry_seq[j] == q; --j) {
      o += w.len[j];
      ++sp;
    }
    w.seq[i] = q;
    w.off[i] = o;
    w.span[i] = sp;
    if (i + 1 == nc || carry_seq[i + 1] != q) {
      w.fills[q] = o + w.len[i];
      w.nspans[q] = sp + 1;
    }
  }
  __syncthreads();

  // ---- C. errors in the reference's order ------------------------------------
  stamp(p, 18);
  const int err_idx = s_misc[1];
  if (tid == 0) {
    p.hdr[MUX_H_N_SEQ] = n_seq;
    p.hdr[MUX_H_ERR_INDEX] = err_idx == INT_MAX ? -1 : err_idx;
  }
  int early = -1;
  if (err_idx != INT_MAX) early = MUX_ERR_PACKING;
  else if (cfg.mode == MUX_MODE_PACK) early = MUX_OK;
  else if (cfg.gbs % (cfg.dp * cfg.mbs) != 0 || cfg.dp * cfg.sp != cfg.world)
    early = MUX_ERR_CONFIG;
  else if (n_seq < cfg.gbs) early = MUX_ERR_VALUE;
  if (early >= 0) {
    emit(cfg, p, w, small, n_seq, false);
    __syncthreads();
    set_status(p, early);
    return;
  }

  // ---- D. batch geometry: cu_seqlens, Ulysses shards, per-rank row bases ------
  stamp(p, 19);
  const int gbs = cfg.gbs, sp = cfg.sp, P = gbs / cfg.dp;
  {
    int64_t carry = 0;
    for (int base = 0; base < gbs; base += nt) {
      const int q = base + tid;
      int64_t tot;
      const int64_t pre = block_excl_scan(q < gbs ? w.fills[q] : 0, &tot, s_warp);
      if (q < gbs) p.cu[q] = (int32_t)(carry + pre);
      carry += tot;
    }
    if (tid == 0) p.cu[gbs] = (int32_t)carry;
  }
  int32_t* s_sstart = reinterpret_cast<int32_t*>(smem + SL.shard);  // [gbs*sp], D..I
  int32_t* s_slen = s_sstart + gbs * sp;
  int32_t* s_cnt = reinterpret_cast<int32_t*>(smem + SL.lpt);       // [gbs*sp], phase E
  int32_t* s_first = s_cnt + gbs * sp;
  for (int x = tid; x < gbs * sp; x += nt) {
    const int q = x / sp, kk = x % sp, F = w.fills[q];
    const int base = F / sp, rem = F % sp;
    const int ln = base + (kk < rem ? 1 : 0);
    const int st = kk * base + (kk < rem ? kk : rem);
    p.shard_len[x] = ln;
    p.shard_start[x] = st;
    s_slen[x] = ln;
    s_sstart[x] = st;
    s_cnt[x] = 0;
    s_first[x] = INT_MAX;
  }
  __syncthreads();
  for (int x = tid; x < W; x += nt) {  // x = r*sp + k
    const int r = x / sp, kk = x % sp;
    int64_t acc = 0;
    for (int j = 0; j < P; ++j) {
      const int q = r * P + j;
      p.row_base[q * sp + kk] = acc;
      acc += s_slen[q * sp + kk];
    }
    p.llm_rows[x] = acc;
  }

  // ---- E. origin rank (owner of the first token), origin_pos ----------------
  stamp(p, 20);
  for (int i = tid; i < S; i += nt) {
    const int q = w.seq[i];
    const int g = group_of_mod(mods[i]);
    w.grp[i] = g;
    if (q < gbs) {
      const int F = w.fills[q];
      int pos = w.off[i];
      if (pos > F - 1) pos = F - 1 > 0 ? F - 1 : 0;
      int kk = 0;
      for (int j = 0; j < sp; ++j)
        if (s_sstart[q * sp + j] <= pos) kk = j;
      w.org[i] = (q / P) * sp + kk;
      w.k[i] = kk;
      atomicAdd(&s_cnt[q * sp + kk], 1);
      atomicMin(&s_first[q * sp + kk], w.span[i]);
    } else {
      w.org[i] = -1;
    }
    w.opos[i] = -1;
    w.enc[i] = -1;
    w.aoff[i] = -1;
    w.eoff[i] = -1;
  }
  __syncthreads();
  for (int x = tid; x < W; x += nt) {  // exclusive prefix of counts within (replica, shard)
    const int r = x / sp, kk = x % sp;
    int acc = 0;
    for (int j = 0; j < P; ++j) {
      const int q = r * P + j;
      const int c = s_cnt[q * sp + kk];
      s_cnt[q * sp + kk] = acc;
      acc += c;
    }
  }
  __syncthreads();
  int nbatch = 0;
  for (int i = tid; i < S; i += nt) {
    const int q = w.seq[i];
    if (q < gbs) {
      const int kk = w.k[i];
      w.opos[i] = s_cnt[q * sp + kk] + w.span[i] - s_first[q * sp + kk];
      ++nbatch;
    }
  }
  {
    int64_t tot;
    block_excl_scan(nbatch, &tot, s_warp);
    if (tid == 0) p.hdr[MUX_H_N_BATCH] = tot;
  }
  auto enc_item = [&](int i) { return w.seq[i] < gbs && w.grp[i] >= 0; };

  // ---- F. loader arena offsets: (origin, group) in table order ----------------
  stamp(p, 21);
  if (tid < kMaxKeys) s_carry[tid] = 0;
  __syncthreads();
  for (int base = 0; base < S; base += nt) {
    const int i = base + tid;
    const bool e = i < S && enc_item(i);
    const int key = e ? w.org[i] * MUX_N_GROUPS + w.grp[i] : -1;
    const int64_t pre = multi_scan(key, e ? w.len[i] : 0, W * MUX_N_GROUPS, s_wk, s_carry);
    if (e) w.aoff[i] = pre;
  }
  for (int x = tid; x < W * MUX_N_GROUPS; x += nt) p.arena_rows[x] = s_carry[x];

  // ---- G. encoder assignment: one sort over (pool, -cost, id, index), then
  //         one warp per pool (LPT), or KK pool by pool.  A pool = (reorder
  //         group of the origin rank, encoder group unless pooled); each pool
  //         is balanced over the RG ranks of its reorder group ----------------
  stamp(p, 22);
  const int ngrp = cfg.pooled ? 1 : MUX_N_GROUPS;
  const int RG = cfg.reorder_group > 0 ? cfg.reorder_group : W;
  const int npools = (W / RG) * ngrp;  // <= 8 * 2 = kMaxKeys
  const int spad = next_pow2(S > 0 ? S : 1);
  double* l_cost = reinterpret_cast<double*>(smem + SL.lpt);
  int64_t* l_id = reinterpret_cast<int64_t*>(l_cost + spad);
  int32_t* l_tidx = reinterpret_cast<int32_t*>(l_id + spad);
  int32_t* l_pool = l_tidx + spad;
  int32_t* l_ord = l_pool + spad;
  int32_t* l_rank = l_ord + spad;
  int32_t* l_org = l_rank + spad;
  int32_t* l_flag = l_org + spad;
  int* s_poff = s_misc + 8;  // pool offsets [npools + 1] (s_misc holds 8 + kMaxKeys + 1)
  auto pool_of = [&](int i) {
    return (w.org[i] / RG) * ngrp + (cfg.pooled ? 0 : w.grp[i]);
  };
  if (tid < kMaxKeys) s_carry[tid] = 0;
  __syncthreads();
  for (int base = 0; base < S; base += nt) {  // position of each encoder item in its pool
    const int i = base + tid;
    const bool e = i < S && enc_item(i);
    const int pool = e ? pool_of(i) : -1;
    const int64_t pre = multi_scan(pool, 1, npools, s_wk, s_carry);
    if (e) w.within[i] = (int32_t)pre;
  }
  if (tid == 0) {
    int acc = 0;
    for (int q = 0; q < npools; ++q) {
      s_poff[q] = acc;
      acc += (int)s_carry[q];
    }
    s_poff[npools] = acc;
  }
  __syncthreads();
  const int m = s_poff[npools];
  for (int i = tid; i < S; i += nt)  // pool-major item order
    if (enc_item(i)) w.order[s_poff[pool_of(i)] + w.within[i]] = i;
  __syncthreads();
  for (int v = tid; v < spad; v += nt) {
    if (v < m) {
      const int i = w.order[v];
      const int q = pool_of(i);
      const double L = (double)w.len[i];
      const int g = w.grp[i];
      // exact in fp64: integer-valued parameters (mux_plan_cfg.cost_model)
      l_cost[v] = cfg.cost_model == MUX_COST_FLOPS
                      ? __dadd_rn(__dmul_rn(cfg.cost_lin[g], L),
                                  __dmul_rn(__dmul_rn(cfg.cost_quad[g], L), L))
                      : L;
      l_id[v] = w.id[i];
      l_tidx[v] = i;
      l_pool[v] = q;
      l_org[v] = w.org[i] - (w.org[i] / RG) * RG;  // origin within its reorder group
    }
    l_ord[v] = v;
  }
  __syncthreads();
  bool kk_overflow = false;
  if (m > 0) {
    if (RG == 1) {
      for (int v = tid; v < m; v += nt) l_rank[v] = 0;
    } else if (cfg.method == MUX_LPT || cfg.method == MUX_LPT_LOCAL ||
               cfg.method == MUX_LPT_LOCAL_RW) {
      bitonic_sort(l_ord, next_pow2(m), PoolKey{l_pool, l_cost, l_id, l_tidx, m});
      const int warp = tid >> 5, nw = nt >> 5;
      for (int q = warp; q < npools; q += nw) {
        const int o = s_poff[q], n = s_poff[q + 1] - o;
        if (n == 0) continue;
        if (cfg.method == MUX_LPT)
          lpt_warp(l_ord + o, l_cost, n, RG, l_rank);
        else
          lpt_local_warp(l_ord + o, l_cost, l_org, n, RG, l_rank, l_flag + o,
                         cfg.method == MUX_LPT_LOCAL_RW);
      }
    } else {
      for (int q = 0; q < npools; ++q) kk_overflow |= s_poff[q + 1] - s_poff[q] > kKkMax;
      if (kk_overflow) {
        if (tid == 0) p.hdr[MUX_H_ERR_INDEX] = -2;  // KK pool limit
      } else {
        KkSmem& K = *reinterpret_cast<KkSmem*>(smem + SL.kk);
        for (int q = 0; q < npools; ++q) {
          const int o = s_poff[q], n = s_poff[q + 1] - o;
          if (tid < 32 && n > 0) kk_warp(K, l_cost + o, n, RG, l_rank + o);
          __syncthreads();
        }
      }
    }
  }
  __syncthreads();
  if (p.hdr[MUX_H_ERR_INDEX] == -2) {
    emit(cfg, p, w, small, n_seq, false);
    __syncthreads();
    set_status(p, MUX_ERR_VALUE);
    return;
  }
  for (int v = tid; v < m; v += nt)  // rank within the group -> world rank
    l_rank[v] += (l_pool[v] / ngrp) * RG;
  __syncthreads();
  for (int v = tid; v < m; v += nt) w.enc[l_tidx[v]] = l_rank[v];
  __syncthreads();

  // ---- H. encoder order = (origin rank, table index); encoder offsets ----------
  stamp(p, 23);
  if (tid < kMaxKeys) s_carry[tid] = 0;
  __syncthreads();
  for (int base = 0; base < S; base += nt) {  // index within origin rank
    const int i = base + tid;
    const bool e = i < S && enc_item(i);
    const int64_t pre = multi_scan(e ? w.org[i] : -1, 1, W, s_wk, s_carry);
    if (e) w.within[i] = (int32_t)pre;
  }
  if (tid == 0) {
    int64_t acc = 0;
    for (int r = 0; r < W; ++r) {
      const int64_t c = s_carry[r];
      s_carry[r] = acc;
      acc += c;
    }
    s_misc[2] = (int)acc;
  }
  __syncthreads();
  for (int i = tid; i < S; i += nt)
    if (enc_item(i)) w.order[s_carry[w.org[i]] + w.within[i]] = i;
  __syncthreads();
  const int n_enc = s_misc[2];
  if (tid < kMaxKeys) s_carry[tid] = 0;
  __syncthreads();
  for (int base = 0; base < n_enc; base += nt) {
    const int t = base + tid;
    const int i = t < n_enc ? w.order[t] : 0;
    const int key = t < n_enc ? w.enc[i] * MUX_N_GROUPS + w.grp[i] : -1;
    const int64_t pre =
        multi_scan(key, t < n_enc ? w.len[i] : 0, W * MUX_N_GROUPS, s_wk, s_carry);
    if (t < n_enc) w.eoff[i] = pre;
  }
  for (int x = tid; x < W * MUX_N_GROUPS; x += nt) p.recv_rows[x] = s_carry[x];
  __syncthreads();

  // ---- H2. staged return (projector, sp == 1): owner-side staging rows per
  //          (owner rank, group), in LLM order = (origin, origin_pos) order ----
  if (cfg.ret_mode == MUX_RET_STAGED) {
    if (tid < kMaxKeys) s_carry[tid] = 0;
    __syncthreads();
    for (int base = 0; base < S; base += nt) {  // batch samples per origin
      const int i = base + tid;
      const bool b = i < S && w.seq[i] < gbs;
      multi_scan(b ? w.org[i] : -1, 1, W, s_wk, s_carry);
    }
    if (tid == 0) {
      int64_t acc = 0;
      for (int r = 0; r < W; ++r) {
        const int64_t c = s_carry[r];
        s_carry[r] = acc;
        acc += c;
      }
      s_misc[2] = (int)acc;
    }
    __syncthreads();
    for (int i = tid; i < S; i += nt)  // w.order <- batch samples by (origin, origin_pos)
      if (w.seq[i] < gbs) w.order[s_carry[w.org[i]] + w.opos[i]] = i;
    __syncthreads();
    const int nb = s_misc[2];
    if (tid < kMaxKeys) s_carry[tid] = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += nt) {
      const int t = base + tid;
      const int i = t < nb ? w.order[t] : 0;
      const bool e = t < nb && w.grp[i] >= 0;
      const int64_t pre = multi_scan(e ? w.org[i] * MUX_N_GROUPS + w.grp[i] : -1,
                                     e ? w.len[i] : 0, W * MUX_N_GROUPS, s_wk, s_carry);
      if (e) p.stage_off[i] = pre;
      else if (t < nb) p.stage_off[i] = -1;
    }
    for (int x = tid; x < W * MUX_N_GROUPS; x += nt) p.stage_rows[x] = s_carry[x];
    __syncthreads();
  }

  // ---- I. LLM positions, return pieces and segment tables of rank `me` -------
  stamp(p, 24);
  const int me = cfg.me;
  auto owner_k = [&](int q, int pos) {
    int kk = 0;
    for (int j = 0; j < sp; ++j)
      if (s_sstart[q * sp + j] <= pos) kk = j;
    return kk;
  };
  const int64_t CH = cfg.chunk_bytes > 0 ? cfg.chunk_bytes : kDefaultChunkBytes;
  int64_t dcarry = 0, rcarry = 0, dchunks = 0, rchunks = 0;
  int64_t dbytes = 0, rbytes = 0, dremote = 0, rremote = 0;
  int64_t gcarry = 0, gchunks = 0, gbytes = 0, gremote = 0;
  int grad_rb[MUX_N_GROUPS];
  for (int q2 = 0; q2 < MUX_N_GROUPS; ++q2)
    grad_rb[q2] = cfg.row_bytes_grad[q2] > 0 ? cfg.row_bytes_grad[q2] : cfg.row_bytes_ret[q2];
  for (int base = 0; base < S; base += nt) {
    const int i = base + tid;
    const bool e = i < S && enc_item(i);
    int npieces = 0, q = 0, L = 0, off = 0, g = 0;
    if (e) {
      q = w.seq[i];
      L = w.len[i];
      off = w.off[i];
      g = w.grp[i];
      const int F = w.fills[q];
      const int k0 = owner_k(q, off < F ? off : (F > 0 ? F - 1 : 0));
      p.llm_rank[i] = (q / P) * sp + k0;
      p.llm_row[i] = p.row_base[q * sp + k0] + off - s_sstart[q * sp + k0];
      if (w.enc[i] == me && L > 0) npieces = owner_k(q, off + L - 1) - owner_k(q, off) + 1;
    } else if (i < S) {
      p.llm_rank[i] = -1;
      p.llm_row[i] = -1;
    }
    const bool disp = e && w.org[i] == me && L > 0;
    int64_t tot, tchk;
    // dispatch segment (one per sample of `me`)
    const int64_t dslot = block_excl_scan(disp ? 1 : 0, &tot, s_warp);
    const int64_t dbytes_i = disp ? (int64_t)L * cfg.row_bytes_in[g] : 0;
    const int64_t dchk_pre = block_excl_scan((dbytes_i + CH - 1) / CH, &tchk, s_warp);
    if (disp) {
      const int64_t v = dcarry + dslot;
      p.dsrc[v] = w.aoff[i];
      p.ddst[v] = w.eoff[i];
      p.drows[v] = L;
      p.dgroup[v] = g;
      p.drank[v] = w.enc[i];
      p.dchunk0[v] = dchunks + dchk_pre;
      dbytes += dbytes_i;
      if (w.enc[i] != me) dremote += dbytes_i;
    }
    dcarry += tot;
    dchunks += tchk;
    // return pieces (one per Ulysses shard the sample touches)
    const int64_t rslot = block_excl_scan(npieces, &tot, s_warp);
    int64_t rchk = 0;
    for (int t = 0; npieces && t < L;) {
      const int pos = off + t, kk = owner_k(q, pos);
      const int end = s_sstart[q * sp + kk] + s_slen[q * sp + kk];
      const int n = (L - t) < (end - pos) ? (L - t) : (end - pos);
      rchk += ((int64_t)n * cfg.row_bytes_ret[g] + CH - 1) / CH;
      t += n;
    }
    const int64_t rchk_pre = block_excl_scan(rchk, &tchk, s_warp);
    int slot = (int)(rcarry + rslot);
    int64_t c0 = rchunks + rchk_pre;
    for (int t = 0; npieces && t < L;) {
      const int pos = off + t, kk = owner_k(q, pos);
      const int end = s_sstart[q * sp + kk] + s_slen[q * sp + kk];
      const int n = (L - t) < (end - pos) ? (L - t) : (end - pos);
      const int dst = (q / P) * sp + kk;
      const int64_t nb = (int64_t)n * cfg.row_bytes_ret[g];
      p.rsrc[slot] = w.eoff[i] + t;
      p.rdst[slot] = cfg.ret_mode == MUX_RET_STAGED
                         ? p.stage_off[i] + t
                         : p.row_base[q * sp + kk] + pos - s_sstart[q * sp + kk];
      p.rrows[slot] = n;
      p.rgroup[slot] = g;
      p.rrank[slot] = dst;
      p.rchunk0[slot] = c0;
      c0 += (nb + CH - 1) / CH;
      rbytes += nb;
      if (dst != me) rremote += nb;
      ++slot;
      t += n;
    }
    rcarry += tot;
    rchunks += tchk;
    // gradient pieces: my LLM rows of this sample, back to its encoder rank
    int gp = 0;
    int64_t gchk = 0;
    for (int t = 0; e && L > 0 && t < L;) {
      const int pos = off + t, kk = owner_k(q, pos);
      const int end = s_sstart[q * sp + kk] + s_slen[q * sp + kk];
      const int n = (L - t) < (end - pos) ? (L - t) : (end - pos);
      if ((q / P) * sp + kk == me) {
        ++gp;
        gchk += ((int64_t)n * grad_rb[g] + CH - 1) / CH;
      }
      t += n;
    }
    const int64_t gslot = block_excl_scan(gp, &tot, s_warp);
    const int64_t gchk_pre = block_excl_scan(gchk, &tchk, s_warp);
    if (gp) {
      int slot2 = (int)(gcarry + gslot);
      int64_t c1 = gchunks + gchk_pre;
      for (int t = 0; t < L;) {
        const int pos = off + t, kk = owner_k(q, pos);
        const int end = s_sstart[q * sp + kk] + s_slen[q * sp + kk];
        const int n = (L - t) < (end - pos) ? (L - t) : (end - pos);
        if ((q / P) * sp + kk == me) {
          const int64_t nb = (int64_t)n * grad_rb[g];
          p.gsrc[slot2] = p.row_base[q * sp + kk] + pos - s_sstart[q * sp + kk];
          p.gdst[slot2] = w.eoff[i] + t;
          p.grows[slot2] = n;
          p.ggroup[slot2] = g;
          p.grank[slot2] = w.enc[i];
          p.gchunk0[slot2] = c1;
          c1 += (nb + CH - 1) / CH;
          gbytes += nb;
          if (w.enc[i] != me) gremote += nb;
          ++slot2;
        }
        t += n;
      }
    }
    gcarry += tot;
    gchunks += tchk;
  }
  {
    int64_t t0, t1, t2, t3, t4, t5;
    block_excl_scan(dbytes, &t0, s_warp);
    block_excl_scan(rbytes, &t1, s_warp);
    block_excl_scan(dremote, &t2, s_warp);
    block_excl_scan(rremote, &t3, s_warp);
    block_excl_scan(gbytes, &t4, s_warp);
    block_excl_scan(gremote, &t5, s_warp);
    if (tid == 0) {
      p.gchunk0[gcarry] = gchunks;
      p.hdr[MUX_H_N_GRAD] = gcarry;
      p.hdr[MUX_H_GRAD_CHUNKS] = gchunks;
      p.hdr[MUX_H_GRAD_BYTES] = t4;
      p.hdr[MUX_H_GRAD_REMOTE] = t5;
      p.dchunk0[dcarry] = dchunks;
      p.rchunk0[rcarry] = rchunks;
      p.hdr[MUX_H_DISPATCH_CHUNKS] = dchunks;
      p.hdr[MUX_H_RETURN_CHUNKS] = rchunks;
      p.hdr[MUX_H_DISPATCH_BYTES] = t0;
      p.hdr[MUX_H_RETURN_BYTES] = t1;
      p.hdr[MUX_H_DISPATCH_REMOTE] = t2;
      p.hdr[MUX_H_RETURN_REMOTE] = t3;
      p.hdr[MUX_H_N_DISPATCH] = dcarry;
      p.hdr[MUX_H_N_RETURN] = rcarry;
      p.hdr[MUX_H_RECV_ROWS0] = p.recv_rows[me * MUX_N_GROUPS + 0];
      p.hdr[MUX_H_RECV_ROWS1] = p.recv_rows[me * MUX_N_GROUPS + 1];
      const bool st = cfg.ret_mode == MUX_RET_STAGED;
      p.hdr[MUX_H_STAGE_ROWS0] = st ? p.stage_rows[me * MUX_N_GROUPS + 0] : 0;
      p.hdr[MUX_H_STAGE_ROWS1] = st ? p.stage_rows[me * MUX_N_GROUPS + 1] : 0;
    }
  }
  emit(cfg, p, w, small, n_seq, true);
  stamp(p, 25);
  __syncthreads();
  set_status(p, MUX_OK);
}

__global__ void __launch_bounds__(kThreads, 1)
    plan_kernel(mux_plan_cfg cfg, const int32_t* lens, const int32_t* mods, const int64_t* ids,
                const int32_t* carry_seq, const int32_t* chunk_off, Plan p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t s_warp[33];
  __shared__ bool s_last;
  if (blockIdx.x == 0) stamp(p, 16);
  if (cfg.n_chunks > 0) ffd_chunk(cfg, lens, ids, chunk_off, p, smem, s_warp);
  // the last CTA to arrive finalises the step
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(p.ticket, 1u);
    s_last = t == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x == 0) *p.ticket = 0;  // re-arm for the next plan
  __threadfence();
  finalize(cfg, lens, mods, ids, carry_seq, chunk_off, p, smem, s_warp);
}

// Stand-alone partition (kk_partition / LPT) of one pool.
__global__ void __launch_bounds__(kThreads, 1) assign_kernel(int method, const double* w,
                                                             const int64_t* ids, int n, int g,
                                                             int32_t* out, const double* init) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int npad = next_pow2(n > 0 ? n : 1);
  double* cost = reinterpret_cast<double*>(smem);
  int64_t* id = reinterpret_cast<int64_t*>(cost + npad);
  int32_t* tidx = reinterpret_cast<int32_t*>(id + npad);
  int32_t* pool = tidx + npad;
  int32_t* ord = pool + npad;
  int32_t* rank = ord + npad;
  for (int k = threadIdx.x; k < npad; k += blockDim.x) {
    if (k < n) {
      cost[k] = w[k];
      id[k] = ids ? ids[k] : k;
      tidx[k] = k;
      pool[k] = 0;
    }
    ord[k] = k;
  }
  __syncthreads();
  if (g == 1) {
    for (int k = threadIdx.x; k < n; k += blockDim.x) rank[k] = 0;
  } else if (method == MUX_LPT) {
    bitonic_sort(ord, npad, PoolKey{pool, cost, id, tidx, n});
    if (threadIdx.x < 32) lpt_warp(ord, cost, n, g, rank, init);
  } else {
    KkSmem& K = *reinterpret_cast<KkSmem*>(smem + align_up(32 * npad, 16));
    if (threadIdx.x < 32) kk_warp(K, cost, n, g, rank);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) out[k] = rank[k];
}

static int plan_smem_bytes(const mux_plan_cfg& c) {
  const int max_seq = c.n_carry_seqs + (c.S - c.n_carry) + 1;
  const int gb = c.mode == MUX_MODE_STEP ? c.gbs * c.sp : 0;
  const SmemPlan SL = smem_plan(c.S, max_seq, gb, c.method);
  int maxn = c.S - c.n_carry;
  int npad = 1;
  while (npad < maxn) npad <<= 1;
  const int ffd = 24 * npad;
  return SL.total > ffd ? SL.total : ffd;
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

static constexpr int kSmemLimit = 227 * 1024 - 10 * 1024;  // leave room for static shared

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
  if (cfg->mode == MUX_MODE_STEP && (cfg->me < 0 || cfg->me >= cfg->world)) {
    set_error("rank %d outside world %d", cfg->me, cfg->world);
    return MUX_ERR_VALUE;
  }
  const int smem = plan_smem_bytes(*cfg);
  if (smem > kSmemLimit) {
    set_error("plan of %d samples needs %d B of shared memory (limit %d)", cfg->S, smem,
              kSmemLimit);
    return MUX_ERR_VALUE;
  }
  static bool attr_done = false;
  if (!attr_done) {
    MUX_CUDA(cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemLimit));
    MUX_CUDA(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemLimit));
    attr_done = true;
  }
  Plan p = make_plan(plan, L);
  const int grid = cfg->n_chunks > 0 ? cfg->n_chunks : 1;
  // Block size follows the step: every phase is a handful of barriers and
  // block scans whose cost grows with the warp count, so small steps (S of a
  // few hundred) run with 4-8 warps.
  int threads = ((cfg->S + 31) / 32) * 32;
  threads = threads < 128 ? 128 : (threads > kThreads ? kThreads : threads);
  plan_kernel<<<grid, threads, smem, static_cast<cudaStream_t>(stream)>>>(
      *cfg, lens, mods, ids, carry_seq, chunk_off, p);
  MUX_CUDA(cudaGetLastError());
  if (cfg->mode == MUX_MODE_STEP && cfg->reshard == MUX_RESHARD_CP_HYBRID)
    return launch_cp_hybrid(*cfg, lens, ids, p, static_cast<cudaStream_t>(stream));
  if (cfg->mode == MUX_MODE_STEP && cfg->lssp_sp > 0)
    return launch_lssp(*cfg, lens, p, static_cast<cudaStream_t>(stream));
  if (cfg->mode == MUX_MODE_STEP && cfg->text_embed)  // text segments from the emitter
    return launch_emit(*cfg, lens, p, 1, INT_MAX, static_cast<cudaStream_t>(stream));
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
      if (h[MUX_H_ERR_INDEX] == -2)
        set_error("encoder pool larger than the KK limit %d", kKkMax);
      else
        set_error("need %d sequences, have %lld", cfg->gbs, (long long)h[MUX_H_N_SEQ]);
      return MUX_ERR_VALUE;
    default:
      set_error("plan did not complete (status %lld)", (long long)st);
      return MUX_ERR_RUNTIME;
  }
}

extern "C" size_t mux_assign_scratch_bytes(int32_t, int32_t) { return 0; }

extern "C" int mux_assign(int32_t method, const double* w, const int64_t* ids, int32_t n,
                          int32_t g, int32_t* out, void* init_loads, void* stream) {
  if (init_loads != nullptr && method != MUX_LPT) {
    set_error("initial loads are only defined for LPT");
    return MUX_ERR_VALUE;
  }
  if (g < 1 || g > 8) {
    set_error("group count %d outside 1..8", g);
    return MUX_ERR_VALUE;
  }
  if (method != MUX_LPT && method != MUX_KK) {
    set_error("stand-alone partition method must be LPT or KK (locality-first LPT needs "
              "origins: use the step planner)");
    return MUX_ERR_VALUE;
  }
  if (n < 0 || n > 4096 || (method == MUX_KK && n > kKkMax)) {
    set_error("%d weights exceed the device limit", n);
    return MUX_ERR_VALUE;
  }
  if (n == 0) return MUX_OK;
  int npad = 1;
  while (npad < n) npad <<= 1;
  const int smem = (int)align_up(32 * npad, 16) + (method == MUX_KK ? (int)sizeof(KkSmem) : 0);
  MUX_CUDA(cudaFuncSetAttribute(assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kSmemLimit));
  assign_kernel<<<1, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      method, w, ids, n, g, out, static_cast<const double*>(init_loads));
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
