// LSSP eta split on the data path (sm_100a): re-targets one step plan so that
// samples longer than eta are encoded in the SP state, sharded over the
// encoder's Ulysses group (SPEC.md:345-353 lssp_schedule).
//
// Runs after plan_kernel on the same stream (one CTA).  It keeps the
// balancer's encoder rank of every sample (its "home"), then
//   * DP samples (len <= eta): whole, on the home rank, compacted to the front
//     of the encoder buffer in encoder order;
//   * SP samples: token shard k (the Ulysses split, first L mod sp shards one
//     token longer) on member k of the home's group, after the DP rows, in
//     (home rank, encoder order);
// and rewrites rank `me`'s dispatch / return / gradient segment tables, their
// chunk maps, the per-rank encoder row counts and the header.  The SP
// all-to-all is fused into the dispatch and return pushes (one hop each), so
// LSSP adds no exchange.  CPU restatement and pinned choices: oracle/lssp.py.

#include "mux_common.cuh"

namespace mux {

namespace {

constexpr int kLsspThreads = 1024;

struct Item {  // staged per sample in shared memory
  int32_t key;  // -1: not encoded; else state << 8 | group << 4 | ... see pack()
  int32_t len;
  int64_t eoff;
};

__device__ __forceinline__ int32_t pack_key(int state, int enc, int grp) {
  return (state << 12) | (enc << 4) | grp;
}
__device__ __forceinline__ int key_state(int32_t k) { return k >> 12; }
__device__ __forceinline__ int key_enc(int32_t k) { return (k >> 4) & 0xff; }
__device__ __forceinline__ int key_grp(int32_t k) { return k & 0xf; }

__device__ __forceinline__ void shard_of(int L, int G, int k, int& s0, int& n) {
  const int b = L / G, r = L % G;
  s0 = k * b + (k < r ? k : r);
  n = b + (k < r ? 1 : 0);
}

// The LLM pieces of batch sample i in token order, f(t0, n, dst_rank, dst_row):
// from the Ulysses shard geometry or, with CpHybrid, the piece table
// reshard.cu wrote.
template <typename F>
__device__ void for_llm_pieces(const mux_plan_cfg& cfg, const Plan& p, int i, int L, F&& f) {
  const int sp = cfg.sp, P = cfg.gbs / cfg.dp;
  const int q = p.seq[i], off = p.off[i];
  if (cfg.reshard == MUX_RESHARD_CP_HYBRID) {
    const int np = p.lp_n[i];
    for (int m = 0; m < np; ++m) {
      const int64_t x = (int64_t)i * sp + m;
      f(p.lp_t0[x], p.lp_len[x], (q / P) * sp + p.lp_k[x], p.lp_row[x]);
    }
    return;
  }
  for (int t = 0; t < L;) {
    const int pos = off + t;
    int kk = 0;
    for (int j = 0; j < sp; ++j)
      if (p.shard_start[q * sp + j] <= pos) kk = j;
    const int end = p.shard_start[q * sp + kk] + p.shard_len[q * sp + kk];
    const int n = (L - t) < (end - pos) ? (L - t) : (end - pos);
    f(t, n, (q / P) * sp + kk, p.row_base[q * sp + kk] + pos - p.shard_start[q * sp + kk]);
    t += n;
  }
}

// Every fragment of sample i (LLM piece x encoder shard), in token order:
// f(t0, n, src_rank, src_row, dst_rank, dst_row).
template <typename F>
__device__ void for_fragments(const mux_plan_cfg& cfg, const Plan& p, int i, int L, int state,
                              int enc, int G, F&& f) {
  const int base = enc - enc % G;
  for_llm_pieces(cfg, p, i, L, [&](int t, int n, int dst, int64_t drow) {
    if (state == 0) {
      f(t, n, enc, p.lssp_row[(int64_t)i * MUX_LSSP_MAX] + t, dst, drow);
    } else {
      for (int k = 0; k < G; ++k) {
        int s0, nk;
        shard_of(L, G, k, s0, nk);
        const int a = t > s0 ? t : s0, b = (t + n) < (s0 + nk) ? (t + n) : (s0 + nk);
        if (a < b)
          f(a, b - a, base + k, p.lssp_row[(int64_t)i * MUX_LSSP_MAX + k] + (a - s0), dst,
            drow + (a - t));
      }
    }
  });
}

__global__ void __launch_bounds__(kLsspThreads, 1)
    lssp_kernel(mux_plan_cfg cfg, const int32_t* __restrict__ lens, Plan p, int G, int eta) {
  extern __shared__ __align__(16) unsigned char smem[];
  Item* it = reinterpret_cast<Item*>(smem);
  __shared__ int64_t s_warp[33];
  __shared__ unsigned long long s_dp[MUX_LSSP_MAX * MUX_N_GROUPS * 1 + 64];
  __shared__ unsigned long long s_sp[MUX_LSSP_MAX * MUX_N_GROUPS * 1 + 64];
  if (p.hdr[MUX_H_STATUS] != MUX_OK) return;  // the plan failed: leave it as is
  const int S = cfg.S, W = cfg.world, me = cfg.me;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int r = tid; r < W * MUX_N_GROUPS; r += nt) s_dp[r] = s_sp[r] = 0;
  // stage: key (state, home, group), length, encoder offset
  for (int i = tid; i < S; i += nt) {
    const int q = p.seq[i], g = p.group[i];
    const bool item = q >= 0 && q < cfg.gbs && g >= 0;
    const int L = lens[i];
    const int state = item ? (L > eta ? 1 : 0) : -1;
    it[i].key = item ? pack_key(state, p.enc[i], g) : -1;
    it[i].len = L;
    it[i].eoff = item ? p.enc_off[i] : 0;
    p.lssp_state[i] = state;
  }
  // token-array offset of every text sample (table order, batch or not)
  if (cfg.text_embed) {
    int64_t carry = 0;
    for (int b0 = 0; b0 < S; b0 += nt) {
      const int i = b0 + tid;
      const bool text = i < S && p.group[i] < 0;
      int64_t tot;
      const int64_t pre = block_excl_scan(text ? lens[i] : 0, &tot, s_warp);
      if (i < S) p.text_off[i] = text ? carry + pre : -1;
      carry += tot;
    }
  }
  __syncthreads();
  // DP rows: compacted in encoder order on the home rank
  for (int i = tid; i < S; i += nt) {
    const int32_t ki = it[i].key;
    if (ki < 0 || key_state(ki) != 0) continue;
    const int64_t ei = it[i].eoff;
    int64_t r = 0;
    for (int j = 0; j < S; ++j)
      if (it[j].key == ki && it[j].eoff < ei) r += it[j].len;
    p.lssp_row[(int64_t)i * MUX_LSSP_MAX] = r;
    atomicAdd(&s_dp[key_enc(ki) * MUX_N_GROUPS + key_grp(ki)], (unsigned long long)it[i].len);
  }
  __syncthreads();
  // SP rows: shard k of every SP sample of the group on member k, after its DP rows
  for (int i = tid; i < S; i += nt) {
    const int32_t ki = it[i].key;
    if (ki < 0 || key_state(ki) != 1) continue;
    const int e = key_enc(ki), g = key_grp(ki), base = e - e % G;
    const int64_t ei = it[i].eoff;
    int64_t r[MUX_LSSP_MAX];
    for (int k = 0; k < G; ++k) r[k] = (int64_t)s_dp[(base + k) * MUX_N_GROUPS + g];
    for (int j = 0; j < S; ++j) {
      const int32_t kj = it[j].key;
      if (kj < 0 || key_state(kj) != 1 || key_grp(kj) != g) continue;
      const int ej = key_enc(kj);
      if (ej - ej % G != base || !(ej < e || (ej == e && it[j].eoff < ei))) continue;
      const int Lj = it[j].len, b = Lj / G, rem = Lj % G;
      for (int k = 0; k < G; ++k) r[k] += b + (k < rem ? 1 : 0);
    }
    const int L = it[i].len;
    for (int k = 0; k < G; ++k) {
      int s0, nk;
      shard_of(L, G, k, s0, nk);
      p.lssp_row[(int64_t)i * MUX_LSSP_MAX + k] = r[k];
      atomicAdd(&s_sp[(base + k) * MUX_N_GROUPS + g], (unsigned long long)nk);
    }
  }
  __syncthreads();
  for (int r = tid; r < W * MUX_N_GROUPS; r += nt)
    p.recv_rows[r] = (int64_t)(s_dp[r] + s_sp[r]);
  // segment tables of rank `me`, in table order (then token order)
  const int64_t CH = cfg.chunk_bytes > 0 ? cfg.chunk_bytes : kDefaultChunkBytes;
  int grad_rb[MUX_N_GROUPS];
  for (int g = 0; g < MUX_N_GROUPS; ++g)
    grad_rb[g] = cfg.row_bytes_grad[g] > 0 ? cfg.row_bytes_grad[g] : cfg.row_bytes_ret[g];
  int64_t tcarry = 0, trows_all = 0;
  int64_t dcarry = 0, rcarry = 0, gcarry = 0, dchunks = 0, rchunks = 0, gchunks = 0;
  int64_t dbytes = 0, rbytes = 0, gbytes = 0, dremote = 0, rremote = 0, gremote = 0;
  for (int b0 = 0; b0 < S; b0 += nt) {
    const int i = b0 + tid;
    int32_t ki = i < S ? it[i].key : -1;
    const int L = i < S ? it[i].len : 0;
    if (L == 0) ki = -1;
    const int state = ki >= 0 ? key_state(ki) : 0, e = ki >= 0 ? key_enc(ki) : 0;
    const int g = ki >= 0 ? key_grp(ki) : 0;
    const int base = e - e % G;
    // dispatch: my loader rows, one segment per shard
    const bool disp = ki >= 0 && p.origin[i] == me;
    int nd = 0;
    int64_t dchk = 0;
    if (disp) {
      const int K = state == 0 ? 1 : G;
      for (int k = 0; k < K; ++k) {
        int s0 = 0, n = L;
        if (state) shard_of(L, G, k, s0, n);
        if (n) {
          ++nd;
          dchk += ((int64_t)n * cfg.row_bytes_in[g] + CH - 1) / CH;
        }
      }
    }
    // return (src == me) and gradient (dst == me) fragments
    int nr = 0, ng = 0;
    int64_t rchk = 0, gchk = 0;
    if (ki >= 0)
      for_fragments(cfg, p, i, L, state, e, G, [&](int, int n, int src, int64_t, int dst, int64_t) {
        if (src == me) {
          ++nr;
          rchk += ((int64_t)n * cfg.row_bytes_ret[g] + CH - 1) / CH;
        }
        if (dst == me) {
          ++ng;
          gchk += ((int64_t)n * grad_rb[g] + CH - 1) / CH;
        }
      });
    int64_t tot, tchk;
    // text rows of `me` (embedding gather, no encoder)
    if (cfg.text_embed) {
      const bool text = i < S && L > 0 && p.group[i] < 0 && p.seq[i] >= 0 && p.seq[i] < cfg.gbs;
      int ntx = 0;
      int64_t nrows = 0;
      if (text)
        for_llm_pieces(cfg, p, i, L, [&](int, int n, int dst, int64_t) {
          if (dst == me) {
            ++ntx;
            nrows += n;
          }
        });
      int64_t ts = tcarry + block_excl_scan(ntx, &tot, s_warp);
      tcarry += tot;
      int64_t tr = trows_all + block_excl_scan(nrows, &tchk, s_warp);
      trows_all += tchk;
      if (ntx)
        for_llm_pieces(cfg, p, i, L, [&](int t, int n, int dst, int64_t drow) {
          if (dst == me) {
            p.tsrc[ts] = p.text_off[i] + t;
            p.tdst[ts] = drow;
            p.trows[ts] = n;
            p.trow0[ts] = tr;
            tr += n;
            ++ts;
          }
        });
    }
    int64_t slot = dcarry + block_excl_scan(nd, &tot, s_warp);
    int64_t c0 = dchunks + block_excl_scan(dchk, &tchk, s_warp);
    dcarry += tot;
    dchunks += tchk;
    if (nd) {
      const int K = state == 0 ? 1 : G;
      const int64_t a = p.arena_off[i];
      for (int k = 0; k < K; ++k) {
        int s0 = 0, n = L;
        if (state) shard_of(L, G, k, s0, n);
        if (!n) continue;
        const int dst = state == 0 ? e : base + k;
        const int64_t nb = (int64_t)n * cfg.row_bytes_in[g];
        p.dsrc[slot] = a + s0;
        p.ddst[slot] = p.lssp_row[(int64_t)i * MUX_LSSP_MAX + (state ? k : 0)];
        p.drows[slot] = n;
        p.dgroup[slot] = g;
        p.drank[slot] = dst;
        p.dchunk0[slot] = c0;
        c0 += (nb + CH - 1) / CH;
        dbytes += nb;
        if (dst != me) dremote += nb;
        ++slot;
      }
    }
    int64_t rslot = rcarry + block_excl_scan(nr, &tot, s_warp);
    int64_t rc0 = rchunks + block_excl_scan(rchk, &tchk, s_warp);
    rcarry += tot;
    rchunks += tchk;
    int64_t gslot = gcarry + block_excl_scan(ng, &tot, s_warp);
    int64_t gc0 = gchunks + block_excl_scan(gchk, &tchk, s_warp);
    gcarry += tot;
    gchunks += tchk;
    if (nr || ng)
      for_fragments(cfg, p, i, L, state, e, G,
                    [&](int, int n, int src, int64_t srow, int dst, int64_t drow) {
                      if (src == me) {
                        const int64_t nb = (int64_t)n * cfg.row_bytes_ret[g];
                        p.rsrc[rslot] = srow;
                        p.rdst[rslot] = drow;
                        p.rrows[rslot] = n;
                        p.rgroup[rslot] = g;
                        p.rrank[rslot] = dst;
                        p.rchunk0[rslot] = rc0;
                        rc0 += (nb + CH - 1) / CH;
                        rbytes += nb;
                        if (dst != me) rremote += nb;
                        ++rslot;
                      }
                      if (dst == me) {
                        const int64_t nb = (int64_t)n * grad_rb[g];
                        p.gsrc[gslot] = drow;
                        p.gdst[gslot] = srow;
                        p.grows[gslot] = n;
                        p.ggroup[gslot] = g;
                        p.grank[gslot] = src;
                        p.gchunk0[gslot] = gc0;
                        gc0 += (nb + CH - 1) / CH;
                        gbytes += nb;
                        if (src != me) gremote += nb;
                        ++gslot;
                      }
                    });
  }
  int64_t t[6];
  block_excl_scan(dbytes, &t[0], s_warp);
  block_excl_scan(rbytes, &t[1], s_warp);
  block_excl_scan(gbytes, &t[2], s_warp);
  block_excl_scan(dremote, &t[3], s_warp);
  block_excl_scan(rremote, &t[4], s_warp);
  block_excl_scan(gremote, &t[5], s_warp);
  if (tid == 0) {
    p.dchunk0[dcarry] = dchunks;
    p.rchunk0[rcarry] = rchunks;
    p.gchunk0[gcarry] = gchunks;
    p.hdr[MUX_H_N_DISPATCH] = dcarry;
    p.hdr[MUX_H_N_RETURN] = rcarry;
    p.hdr[MUX_H_N_GRAD] = gcarry;
    p.hdr[MUX_H_DISPATCH_CHUNKS] = dchunks;
    p.hdr[MUX_H_RETURN_CHUNKS] = rchunks;
    p.hdr[MUX_H_GRAD_CHUNKS] = gchunks;
    p.hdr[MUX_H_DISPATCH_BYTES] = t[0];
    p.hdr[MUX_H_RETURN_BYTES] = t[1];
    p.hdr[MUX_H_GRAD_BYTES] = t[2];
    p.hdr[MUX_H_DISPATCH_REMOTE] = t[3];
    p.hdr[MUX_H_RETURN_REMOTE] = t[4];
    p.hdr[MUX_H_GRAD_REMOTE] = t[5];
    p.hdr[MUX_H_N_TEXT] = cfg.text_embed ? tcarry : 0;
    p.hdr[MUX_H_TEXT_ROWS] = cfg.text_embed ? trows_all : 0;
    if (cfg.text_embed) p.trow0[tcarry] = trows_all;
    p.hdr[MUX_H_RECV_ROWS0] = (int64_t)(s_dp[me * MUX_N_GROUPS] + s_sp[me * MUX_N_GROUPS]);
    p.hdr[MUX_H_RECV_ROWS1] =
        (int64_t)(s_dp[me * MUX_N_GROUPS + 1] + s_sp[me * MUX_N_GROUPS + 1]);
  }
}

}  // namespace

// Segment tables for encoder groups of G ranks and threshold eta (G = 1 and
// eta = INT_MAX: every sample DP, i.e. the plain encoder layout).
int launch_emit(const mux_plan_cfg& cfg, const int32_t* lens, const Plan& p, int G, int eta,
                cudaStream_t stream) {
  const int smem = (cfg.S > 0 ? cfg.S : 1) * (int)sizeof(Item);
  static bool attr = false;
  if (!attr) {
    MUX_CUDA(cudaFuncSetAttribute(lssp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  4096 * (int)sizeof(Item)));
    attr = true;
  }
  int threads = ((cfg.S + 31) / 32) * 32;
  threads = threads < 128 ? 128 : (threads > kLsspThreads ? kLsspThreads : threads);
  lssp_kernel<<<1, threads, smem, stream>>>(cfg, lens, p, G, eta);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

int launch_lssp(const mux_plan_cfg& cfg, const int32_t* lens, const Plan& p, cudaStream_t stream) {
  return launch_emit(cfg, lens, p, cfg.lssp_sp, cfg.lssp_eta, stream);
}

}  // namespace mux
