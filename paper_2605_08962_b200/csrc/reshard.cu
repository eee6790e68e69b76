// CpHybrid LLM placement on the data path (sm_100a): reshard.plan_reshard's
// CpHybrid variant (§5.2 "only shard long
// samples") applied to one step plan.
//
// Runs after plan_kernel on the same stream, one CTA, one warp per batch
// sequence.  In the replica's CP group of sp ranks, samples longer than
// cp_threshold (0: capacity / sp) are split sp ways (first L mod sp pieces one
// token longer); the others stay whole and go by LPT — order (-len, id, span
// index), least-loaded rank, lowest rank on ties — onto the loads the long
// pieces left.  On CP rank k the rows of sequence q are the
// pieces k holds, in span order, and the replica's sequences follow each
// other.  The kernel writes the per-sample piece table, each (sequence, k)
// load (shard_len) and first row (row_base), llm_rows and llm_rank/llm_row;
// the segment tables then come from lssp.cu's emitter.  CPU restatement:
// oracle/cphybrid.py.

#include <climits>

#include "mux_common.cuh"

namespace mux {

namespace {

constexpr int kCphThreads = 1024;

__global__ void __launch_bounds__(kCphThreads, 1)
    cph_kernel(mux_plan_cfg cfg, const int32_t* __restrict__ lens,
               const int64_t* __restrict__ ids, Plan p) {
  extern __shared__ __align__(16) unsigned char smem[];
  int32_t* cuspan = reinterpret_cast<int32_t*>(smem);  // [gbs + 1]
  int32_t* sidx = cuspan + cfg.gbs + 1;                // [S]: sample of (sequence, span)
  __shared__ int64_t s_warp[33];
  if (p.hdr[MUX_H_STATUS] != MUX_OK) return;
  const int S = cfg.S, gbs = cfg.gbs, sp = cfg.sp, P = cfg.gbs / cfg.dp;
  const int thr = cfg.cp_threshold > 0 ? cfg.cp_threshold : cfg.capacity / sp;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = nt >> 5;
  // span-ordered sample index of every batch sequence
  int64_t carry = 0;
  for (int b0 = 0; b0 < gbs; b0 += nt) {
    const int q = b0 + tid;
    const int64_t v = q < gbs ? p.nspans[q] : 0;
    int64_t tot;
    const int64_t pre = block_excl_scan(v, &tot, s_warp);
    if (q < gbs) cuspan[q] = (int32_t)(carry + pre);
    carry += tot;
  }
  if (tid == 0) cuspan[gbs] = (int32_t)carry;
  __syncthreads();
  for (int i = tid; i < S; i += nt) {
    const int q = p.seq[i];
    if (q >= 0 && q < gbs) sidx[cuspan[q] + p.span[i]] = i;
  }
  __syncthreads();
  int32_t* ord = p.scratch_a;   // LPT order of the short samples, per sequence
  int32_t* rank_of = p.scratch_b;  // CP rank index of each short sample
  for (int q = warp; q < gbs; q += nwarps) {
    const int b = cuspan[q], n = cuspan[q + 1] - b;
    // loads of the long pieces (lane k holds rank k's load)
    int load = 0;
    for (int j = 0; j < n; ++j) {
      const int L = lens[sidx[b + j]];
      if (L > thr && lane < sp) load += L / sp + (lane < L % sp ? 1 : 0);
    }
    // LPT order of the short samples: rank by (-len, id, span index)
    int nshort = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + lane;
      const bool sh = j < n && lens[sidx[b + j]] <= thr;
      nshort += __popc(__ballot_sync(MUX_FULL, sh));
      if (!sh) continue;
      const int i = sidx[b + j], L = lens[i];
      const int64_t id = ids[i];
      int r = 0;
      for (int jj = 0; jj < n; ++jj) {
        const int ii = sidx[b + jj], LL = lens[ii];
        if (LL > thr) continue;
        const int64_t idd = ids[ii];
        if (LL > L || (LL == L && (idd < id || (idd == id && jj < j)))) ++r;
      }
      ord[b + r] = j;
    }
    __syncwarp();
    for (int r = 0; r < nshort; ++r) {
      const int i = sidx[b + ord[b + r]];
      const int key = lane < sp ? load * 64 + lane : INT_MAX;
      const int k = __reduce_min_sync(MUX_FULL, key) & 63;
      if (lane == k) load += lens[i];
      if (lane == 0) rank_of[i] = k;
    }
    __syncwarp();
    if (lane < sp) p.shard_len[q * sp + lane] = load;
    // pieces in span order, rows local to (q, k)
    if (lane == 0) {
      int off[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int j = 0; j < n; ++j) {
        const int i = sidx[b + j], L = lens[i];
        const int64_t x0 = (int64_t)i * sp;
        int np = 0;
        if (L > thr) {
          for (int k = 0; k < sp; ++k) {
            const int bq = L / sp, rem = L % sp;
            const int s0 = k * bq + (k < rem ? k : rem), nk = bq + (k < rem ? 1 : 0);
            if (nk > 0) {
              p.lp_k[x0 + np] = k;
              p.lp_t0[x0 + np] = s0;
              p.lp_len[x0 + np] = nk;
              p.lp_row[x0 + np] = off[k];
              ++np;
            }
            off[k] += nk;
          }
        } else {
          const int k = rank_of[i];
          if (L > 0) {
            p.lp_k[x0] = k;
            p.lp_t0[x0] = 0;
            p.lp_len[x0] = L;
            p.lp_row[x0] = off[k];
            np = 1;
          }
          off[k] += L;
        }
        p.lp_n[i] = np;
      }
    }
  }
  __syncthreads();
  // first row of each (sequence, k) on its rank; rows per LLM rank
  for (int t = tid; t < cfg.dp * sp; t += nt) {
    const int r = t / sp, k = t % sp;
    int64_t acc = 0;
    for (int q = r * P; q < (r + 1) * P; ++q) {
      p.row_base[q * sp + k] = acc;
      acc += p.shard_len[q * sp + k];
    }
    p.llm_rows[r * sp + k] = acc;
  }
  __syncthreads();
  for (int i = tid; i < S; i += nt) {
    const int q = p.seq[i];
    if (q < 0 || q >= gbs) continue;
    const int np = p.lp_n[i];
    for (int m = 0; m < np; ++m) {
      const int64_t x = (int64_t)i * sp + m;
      p.lp_row[x] += p.row_base[q * sp + p.lp_k[x]];
    }
    if (p.group[i] >= 0) {
      p.llm_rank[i] = np ? (q / P) * sp + p.lp_k[(int64_t)i * sp] : -1;
      p.llm_row[i] = np ? p.lp_row[(int64_t)i * sp] : -1;
    }
  }
}

}  // namespace

int launch_cp_hybrid(const mux_plan_cfg& cfg, const int32_t* lens, const int64_t* ids,
                     const Plan& p, cudaStream_t stream) {
  const int smem = (cfg.gbs + 1 + (cfg.S > 0 ? cfg.S : 1)) * 4;
  cph_kernel<<<1, kCphThreads, smem, stream>>>(cfg, lens, ids, p);
  MUX_CUDA(cudaGetLastError());
  const bool lssp = cfg.lssp_sp > 0;
  return launch_emit(cfg, lens, p, lssp ? cfg.lssp_sp : 1, lssp ? cfg.lssp_eta : INT_MAX, stream);
}

}  // namespace mux
