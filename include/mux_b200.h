/*
 * mux_b200.h — C ABI of libmuxb200.so, the B200 data path between modality
 * encoders and the LLM backbone (arXiv 2605.08962 / reference package muxsim).
 *
 * Plain C: device pointers, sizes and a cudaStream_t passed as void*.  The
 * library never allocates or frees caller memory; every buffer is owned by the
 * caller (PyTorch on the Python side).  Status codes map one-to-one onto the
 * reference's exception types (pkg/src/muxsim/workload.py:29-34):
 *   MUX_ERR_CONFIG  -> ConfigError      MUX_ERR_PACKING -> PackingError
 *   MUX_ERR_VALUE   -> ValueError       MUX_ERR_RUNTIME -> RuntimeError
 * and mux_last_error() returns the thread-local message.
 *
 * Reference interfaces each entry point replaces (file:line under
 * /root/reference):
 *   mux_plan_step        workload.hybrid_pack (pkg/src/muxsim/workload.py:240-262)
 *                        + build_global_batch (:265-278) + replica slicing
 *                        (:177-180) + balance.grouped_reorder / kk_partition
 *                         + reshard.plan_reshard UlyssesUniform
 *                        (SPEC.md:462-470), fused into one device plan; with
 *                        cfg.reshard = CpHybrid, plan_reshard's CpHybrid variant
 *                        (SPEC.md:456-469, :497); with cfg.lssp_sp, the LSSP
 *                        eta split of lssp_schedule; with
 *                        cfg.text_embed, the text rows' segment table.
 *   mux_assign           balance.kk_partition and the LPT
 *                        greedy named by BASELINE.json north_star.
 *   mux_segcopy          the data all-to-all of grouped_reorder
 *                        and the inverse of restore_order;
 *                        pack, dispatch, return and scatter are all segment
 *                        copies over local or NVLink-peer pointers.
 *   mux_signal/mux_wait  cross-GPU completion flags for the push exchange.
 *   mux_proj_scatter*    projector GEMM fused with the placeholder scatter
 *                        (no reference code, adapter); the
 *                        grouped forms run both encoder groups in one launch
 *                        and can fuse the completion signal.
 *   mux_text_embed       the LLM embedding rows of the text tokens in the same
 *                        packed buffer.
 *   mux_encoder_standin  deterministic stand-in for the (out of scope) encoder.
 */
#ifndef MUX_B200_H
#define MUX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MUX_OK 0
#define MUX_ERR_CONFIG 1
#define MUX_ERR_PACKING 2
#define MUX_ERR_VALUE 3
#define MUX_ERR_CUDA 4
#define MUX_ERR_RUNTIME 5

#define MUX_MODE_PACK 0 /* FFD only: hybrid_pack of each chunk              */
#define MUX_MODE_STEP 1 /* full step: batch, origins, balance, reshard, segs */

#define MUX_LPT 0
#define MUX_KK 1
#define MUX_LPT_LOCAL 2 /* locality-first LPT: keep samples on their origin rank up to
                           the balanced load, LPT the rest on top */
#define MUX_LPT_LOCAL_RW 3 /* as MUX_LPT_LOCAL, but pass 2 charges a sample 9/8 of its
                              cost on a rank other than its origin (NVLink-moved rows) */

#define MUX_N_GROUPS 2 /* encoder groups: 0 = vision (image/video), 1 = audio */

/* Header slots of the plan buffer (int64 each). */
#define MUX_H_STATUS 0
#define MUX_H_ERR_INDEX 1     /* table index of the first oversize sample, -1  */
#define MUX_H_N_SEQ 2         /* sequences after packing (carry + new)         */
#define MUX_H_N_DISPATCH 3    /* dispatch segments of rank `me`                */
#define MUX_H_N_RETURN 4      /* return pieces of rank `me`                    */
#define MUX_H_DISPATCH_CHUNKS 5
#define MUX_H_RETURN_CHUNKS 6
#define MUX_H_DISPATCH_BYTES 7
#define MUX_H_RETURN_BYTES 8
#define MUX_H_N_BATCH 9       /* samples inside the global batch               */
#define MUX_H_DISPATCH_REMOTE 10 /* dispatch bytes leaving rank `me`           */
#define MUX_H_RETURN_REMOTE 11   /* return bytes leaving rank `me`             */
#define MUX_H_RECV_ROWS0 12   /* rows received by `me`, group 0 / group 1      */
#define MUX_H_RECV_ROWS1 13
#define MUX_H_STAGE_ROWS0 14  /* rows staged on `me` for its projector, group 0/1 */
#define MUX_H_STAGE_ROWS1 15
#define MUX_H_N_GRAD 16      /* gradient-return pieces of rank `me` (LLM owner)  */
#define MUX_H_GRAD_CHUNKS 17
#define MUX_H_GRAD_BYTES 18
#define MUX_H_GRAD_REMOTE 19
#define MUX_H_STAMP0 20      /* 20..29: planner phase timestamps (globaltimer)  */
#define MUX_H_N_TEXT 30      /* text segments of rank `me` (cfg.text_embed)      */
#define MUX_H_TEXT_ROWS 31   /* text rows of rank `me`                          */
#define MUX_H_SLOTS 32

#define MUX_RET_FINAL 0  /* return rows go to their final packed-LLM rows           */
#define MUX_RET_STAGED 1 /* return d_enc rows to the owner's per-group staging      */
                         /* buffer (LLM order); the owner then projects locally     */

typedef struct {
  int32_t S;            /* samples in the step table                        */
  int32_t n_carry;      /* leading carry samples (sequence/span order)      */
  int32_t n_carry_seqs; /* carried sequences                                */
  int32_t n_chunks;     /* drawn chunks after the carry samples             */
  int32_t capacity;
  int32_t gbs, dp, sp, world, mbs;
  int32_t method;       /* MUX_LPT | MUX_KK | MUX_LPT_LOCAL                 */
  int32_t pooled;       /* 1: balance all modalities together */
  int32_t me;           /* rank whose segment tables are emitted            */
  int32_t mode;         /* MUX_MODE_PACK | MUX_MODE_STEP                    */
  int32_t row_bytes_in[MUX_N_GROUPS];  /* loader row bytes per group        */
  int32_t row_bytes_ret[MUX_N_GROUPS]; /* returned row bytes per group      */
  int32_t chunk_bytes;  /* copy work unit (0 = default 32 KiB)              */
  int32_t ret_mode;     /* MUX_RET_FINAL | MUX_RET_STAGED (sp == 1 only)      */
  int32_t row_bytes_grad[MUX_N_GROUPS]; /* gradient-return row bytes (0: = ret) */
  /* LSSP eta split: lssp_sp = encoder Ulysses group size
   * (1..MUX_LSSP_MAX, divides world; 0 = off); samples longer than lssp_eta
   * are encoded in the SP state, one token shard per group member. */
  int32_t lssp_sp, lssp_eta;
  /* LLM-side placement (reshard.plan_reshard): Ulysses
   * uniform shards (default) or CpHybrid over the replica's sp ranks (long
   * samples, len > cp_threshold, split sp ways; short ones whole by LPT on the
   * residual loads).  cp_threshold 0 = capacity / sp. */
  int32_t reshard, cp_threshold;
  /* 1: also emit rank `me`'s text segments (token offset -> LLM row) so
   * mux_text_embed can gather the text tokens' embedding rows into the same
   * packed LLM buffer. */
  int32_t text_embed;
  /* Reorder groups (SPEC.md:383 ReorderGroup, :208 reorder_group_size):
   * consecutive blocks of reorder_group ranks; a sample is balanced only over
   * the ranks of its origin rank's group (0 = the whole world). */
  int32_t reorder_group;
  /* Per-sample balancing cost (SPEC.md:390 token counts by default; the
   * optional encoder cost of costs.flops_forward, costs.py:108-124):
   * MUX_COST_TOKENS: cost = len;  MUX_COST_FLOPS: cost = cost_lin[g] * len +
   * cost_quad[g] * len * len for encoder group g, i.e. flops_forward with
   * cost_lin = 2 P, cost_quad = 2 layers hidden (encoder seq_len = len), mult 1.
   * Integer-valued parameters keep every cost and load sum exact in fp64
   * (bit-identical plans on every rank) while the sums stay below 2^50. */
  int32_t cost_model;
  int32_t reserved0;
  double cost_lin[MUX_N_GROUPS];
  double cost_quad[MUX_N_GROUPS];
} mux_plan_cfg;

#define MUX_COST_TOKENS 0
#define MUX_COST_FLOPS 1

#define MUX_RESHARD_ULYSSES 0
#define MUX_RESHARD_CP_HYBRID 1

#define MUX_LSSP_MAX 8

/* Byte offsets of every array inside the plan buffer (one device blob). */
typedef struct {
  int64_t header;                                   /* int64[MUX_H_SLOTS] */
  int64_t sync;     /* uint32 ticket; must be zero when the blob is first used */
  int64_t seq, off, span, origin, origin_pos, group, enc; /* int32[S]      */
  int64_t arena_off, enc_off, stage_off;            /* int64[S]           */
  int64_t llm_rank, llm_row;                        /* int32/int64[S]     */
  int64_t bin_fill, bin_nspan, bin_of;              /* int32[S] (scratch) */
  int64_t chunk_nbins, chunk_err;                   /* int32[n_chunks]    */
  int64_t fills, nspans;                            /* int32[max_seq]     */
  int64_t cu;                                       /* int32[gbs+1]       */
  int64_t shard_len, shard_start;                   /* int32[gbs*sp]      */
  int64_t row_base;                                 /* int64[gbs*sp]      */
  int64_t arena_rows, recv_rows, stage_rows;        /* int64[world*2]     */
  int64_t llm_rows;                                 /* int64[world]       */
  int64_t order, scratch_a, scratch_b;              /* int32[S] (scratch) */
  /* dispatch segments (rank me): rows from arena[group] to recv[group]@enc */
  int64_t dseg_src_row, dseg_dst_row, dseg_rows;    /* int64[S]           */
  int64_t dseg_group, dseg_dst_rank;                /* int32[S]           */
  int64_t dseg_chunk0;  /* int64[S+1]: first copy chunk of each segment   */
  /* return pieces (rank me): rows from enc_out[group] to llm@dst_rank      */
  int64_t rseg_src_row, rseg_dst_row, rseg_rows;    /* int64[S*(sp+1)]    */
  int64_t rseg_group, rseg_dst_rank;                /* int32[S*(sp+1)]    */
  int64_t rseg_chunk0;                              /* int64[S*(sp+1)+1]  */
  /* gradient return (rank me as LLM owner): dY rows at my LLM rows back to
   * their encoder rank's gradient buffer in encoder order     */
  int64_t gseg_src_row, gseg_dst_row, gseg_rows;    /* int64[S*(sp+1)]    */
  int64_t gseg_group, gseg_dst_rank;                /* int32[S*(sp+1)]    */
  int64_t gseg_chunk0;                              /* int64[S*(sp+1)+1]  */
  /* LSSP (lssp_sp > 0): state per sample (0 DP, 1 SP, -1 not encoded) and
   * encoder-buffer row per (sample, shard): DP in column 0 on the home rank,
   * SP shard k on group member k.  With LSSP the dispatch table holds up to
   * S*lssp_sp segments and the return/gradient tables S*(sp+1+lssp_sp). */
  int64_t lssp_state;                               /* int32[S]           */
  int64_t lssp_row;                                 /* int64[S*MUX_LSSP_MAX] */
  /* CpHybrid LLM pieces per sample (reshard == MUX_RESHARD_CP_HYBRID): count,
   * then per piece the CP rank index k, first token, tokens and LLM row on
   * rank (replica * sp + k).  shard_len then holds each (sequence, k) load
   * and row_base its first row. */
  int64_t lp_n;                                     /* int32[S]           */
  int64_t lp_k, lp_t0, lp_len;                      /* int32[S*sp]        */
  int64_t lp_row;                                   /* int64[S*sp]        */
  /* text rows (cfg.text_embed): token-array offset of every text sample
   * (table order over all text samples), then rank `me`'s text segments and
   * their row prefix (tseg_row0[n] = total rows). */
  int64_t text_off;                                 /* int64[S]           */
  int64_t tseg_src, tseg_dst, tseg_rows;            /* int64[S*(sp+1)]    */
  int64_t tseg_row0;                                /* int64[S*(sp+1)+1]  */
  int64_t total;
} mux_plan_layout;

int mux_version(void);
/* sizeof(mux_plan_cfg), sizeof(mux_plan_layout), sizeof(mux_proj_group) into
 * out[0..2]: lets a binding check its struct mirrors against this build. */
void mux_abi_sizes(int64_t* out);
const char* mux_last_error(void);

/* Layout of the plan buffer for `cfg`; returns MUX_OK or MUX_ERR_VALUE. */
int mux_plan_layout_of(const mux_plan_cfg* cfg, mux_plan_layout* out);

/* One device plan for one step (or, in MUX_MODE_PACK, FFD of each chunk).
 * Table arrays are device pointers: lens/mods int32[S], ids int64[S],
 * carry_seq int32[n_carry], chunk_off int32[n_chunks+1] (chunk_off[0] =
 * n_carry).  Stream-ordered; errors are written to the header and reported
 * by mux_plan_check() after the caller synchronises. */
int mux_plan_step(const mux_plan_cfg* cfg, const int32_t* lens, const int32_t* mods,
                  const int64_t* ids, const int32_t* carry_seq, const int32_t* chunk_off,
                  void* plan, size_t plan_bytes, void* stream);

/* Host-side check of a plan header copied back by the caller: maps the
 * device status onto MUX_ERR_* and sets mux_last_error() with the
 * reference's message. `ids_host`/`lens_host` name the offender. */
int mux_plan_check(const mux_plan_cfg* cfg, const int64_t* header_host,
                   const int64_t* ids_host, const int32_t* lens_host);

/* Stand-alone partition of n weights over g ranks (kk_partition / LPT).
 * weights double[n], ids int64[n] (LPT tie-break; NULL = index), out int32[n],
 * init_loads double[g] (LPT only: loads the ranks start with, e.g. the
 * residual capacity rule of CpHybrid; NULL = zeros).  Device
 * pointers. */
size_t mux_assign_scratch_bytes(int32_t n, int32_t g);
int mux_assign(int32_t method, const double* weights, const int64_t* ids, int32_t n,
               int32_t g, int32_t* out, void* init_loads, void* stream);

/* Segment copy: table = plan (dispatch: which=0, return: which=1,
 * gradient return: which=2 with src_bases[group] = the dY buffer (LLM rows,
 * row_bytes_ret wide) and dst_bases[rank * MUX_N_GROUPS + group]).
 * src_bases[group], dst_bases[rank * MUX_N_GROUPS + group] (dispatch) or
 * dst_bases[rank] (return) are device arrays of device pointers (local or
 * NVLink-peer).  Row bytes come from the plan cfg.  CTAs grab chunks from a
 * device counter: `sync` is uint32[2] in device memory, zero before the first
 * launch and re-armed by the kernel.  grid_ctas = 0 picks the persistent
 * default (SMs x occupancy). */
int mux_segcopy(const mux_plan_cfg* cfg, const void* plan, int32_t which,
                void* const* src_bases, void* const* dst_bases, int32_t grid_ctas,
                uint32_t* sync, void* stream);
/* Same copy, then the last CTA advances the device epoch counter
 * (e = ++*epoch_ctr), fences at system scope and stores e into
 * flags_peers[r][me] for every rank r (fused completion signal).  Epochs live
 * in device memory, so a captured CUDA graph of the step replays correctly. */
int mux_segcopy_signal(const mux_plan_cfg* cfg, const void* plan, int32_t which,
                       void* const* src_bases, void* const* dst_bases, int32_t grid_ctas,
                       uint64_t* const* flags_peers, uint32_t* sync, uint64_t* epoch_ctr,
                       void* stream);

/* General form: segments whose destination rank is `skip_rank` are not
 * copied (-1: copy all); flags_peers may be NULL (no completion signal).
 * grid_ctas < 0 launches -grid_ctas CTAs without shared memory, so the copy
 * can co-reside with a kernel that holds the SMs' shared memory.
 * poison (nullable): the path's device status word, the err_dev of its
 * mux_wait calls.  Nonzero = the step is poisoned (a flag wait timed out or
 * saw a poisoned peer): the copy moves nothing and publishes its epoch with
 * MUX_POISON_BIT set, so every peer's wait fails fast too. */
int mux_segcopy_ex(const mux_plan_cfg* cfg, const void* plan, int32_t which,
                   void* const* src_bases, void* const* dst_bases, int32_t grid_ctas,
                   int32_t skip_rank, uint64_t* const* flags_peers, uint32_t* sync,
                   uint64_t* epoch_ctr, const int32_t* poison, void* stream);

/* One contiguous 8-byte-aligned byte range with the same copy engine as
 * mux_segcopy (local or NVLink-peer dst/src); used by the NVLink probe. */
int mux_copy_bytes(void* dst, const void* src, int64_t n, int32_t grid_ctas, void* stream);
/* n byte ranges (device arrays dsts/srcs/bytes; max_bytes = the longest, known
 * to the caller) in one launch, 32 KiB chunks dealt round-robin over the
 * ranges so every destination is written concurrently.  mode 0: SM
 * loads/stores (the segment-copy engine); mode 1: TMA bulk copies through
 * shared memory (cp.async.bulk); ranges 16-byte aligned for mode 1.  The
 * NVLink probe's all-to-all and engine A/B. */
int mux_copy_ranges(int32_t n, void* const* dsts, const void* const* srcs, const int64_t* bytes,
                    int64_t max_bytes, int32_t grid_ctas, int32_t mode, void* stream);
/* cudaMemcpyAsync(cudaMemcpyDefault): the copy-engine comparator of the probe. */
int mux_memcpy_async(void* dst, const void* src, int64_t n, void* stream);

/* Cross-GPU completion flags.  flags_peers: device array of `world` device
 * pointers to each rank's uint64 flag array (world entries each).  signal
 * advances the device epoch counter (e = ++*epoch_ctr) and stores e into
 * flag[me] of every peer after a system-scope fence; wait spins until every
 * flag[src] of `my_flags` >= *epoch_ctr (bounded: timeout_ms; a timeout sets
 * *err_dev = 1 and returns; a flag carrying MUX_POISON_BIT sets *err_dev = 2;
 * a wait issued while *err_dev != 0 returns at once). */
#define MUX_POISON_BIT (1ull << 63)
int mux_signal(int32_t me, int32_t world, uint64_t* const* flags_peers, uint64_t* epoch_ctr,
               void* stream);
int mux_wait(int32_t world, const uint64_t* my_flags, const uint64_t* epoch_ctr,
             int32_t timeout_ms, int32_t* err_dev, void* stream);
/* mux_wait for an explicit epoch (known to the host) instead of the value of
 * this rank's own counter — for a wait issued on a stream that does not
 * follow the signalling launch. */
int mux_wait_value(int32_t world, const uint64_t* my_flags, uint64_t target, int32_t timeout_ms,
                   int32_t* err_dev, void* stream);
/* mux_signal with fence = 0: no system-scope fence before the flag stores.
 * For a permission signal ("my buffer may be overwritten") issued after
 * kernels that only read that buffer: stream order already completed them. */
int mux_signal_ex(int32_t me, int32_t world, uint64_t* const* flags_peers, uint64_t* epoch_ctr,
                  int32_t fence, void* stream);

/* Deterministic encoder stand-in: for every sample of rank `me` in group
 * `group`, rows [enc_off, enc_off+len) of out (row width `width` bf16)
 * get E(id, t, c).  Uses the plan's enc/enc_off/group arrays. */
int mux_encoder_standin(const mux_plan_cfg* cfg, const void* plan, const int64_t* ids,
                        const int32_t* lens, int32_t group, int32_t width,
                        uint16_t* out, void* stream);

/* Expand return pieces of rank `me`, group `group` into a per-row
 * destination table: row_dst[src_row] = (dst_rank << 40) | dst_row.
 * group = -1: every group in one launch, group g's table at
 * row_dst + g * n_rows. */
int mux_return_rows(const mux_plan_cfg* cfg, const void* plan, int32_t group,
                    int64_t* row_dst, int64_t n_rows, void* stream);

/* MUX_RET_STAGED: per-row destination of the owner's staging rows of
 * `group`: row_dst[stage_off + t] = (me << 40) | (llm_row + t).  lens: the
 * step table's int32 lengths (device). */
int mux_stage_rows(const mux_plan_cfg* cfg, const void* plan, const int32_t* lens,
                   int32_t group, int64_t* row_dst, int64_t n_rows, void* stream);

/* Text rows of the packed LLM input: for every text segment of rank `me`
 * (plan made with cfg.text_embed = 1), out[dst_row + t, :] =
 * table[tokens[src + t], :], t < rows.  tokens: int32 token ids of the
 * step's text samples in table order (text_off); table: bf16 [vocab, d]
 * embedding rows, replicated on every LLM rank; out: this rank's packed LLM
 * buffer (row stride d).  Ids outside [0, vocab) are skipped and counted in
 * *err (device int32).  d % 8 == 0. */
int mux_text_embed(const mux_plan_cfg* cfg, const void* plan, const int32_t* tokens,
                   const uint16_t* table, int64_t vocab, int32_t d, uint16_t* out, int32_t* err,
                   void* stream);

/* Projector fused with the scatter: for m < M,
 *   out_rank[row_dst[m] >> 40][row_dst[m] & (2^40-1), :] =
 *       bf16( X[m, :K] . W[:N, :K]^T + bias[:N] )
 * X bf16 [M, K] row-major, W bf16 [N, K] row-major (nn.Linear weight),
 * bias bf16 [N] or NULL, out_bases: device array of world device pointers
 * (local or NVLink-peer LLM buffers, row stride N).  tcgen05 + TMEM + TMA
 * on sm_100a.  K % 64 == 0, N % 256 == 0. */
int mux_proj_scatter(const uint16_t* X, const uint16_t* W, const uint16_t* bias, int64_t M,
                     int32_t K, int32_t N, const int64_t* row_dst, void* const* out_bases,
                     int32_t num_sms, void* stream);

/* Same, with the row count read from device memory at launch (*M_dev,
 * clamped to M_max) so the step needs no host sync; M_max bounds X. */
int mux_proj_scatter_dev(const uint16_t* X, const uint16_t* W, const uint16_t* bias,
                         int64_t M_max, const int64_t* M_dev, int32_t K, int32_t N,
                         const int64_t* row_dst, void* const* out_bases, int32_t num_sms,
                         void* stream);

/* One projector problem of a grouped launch (one per encoder group). */
typedef struct {
  const uint16_t* X;       /* bf16 [M_max, K] encoder rows                     */
  const uint16_t* W;       /* bf16 [N, K] nn.Linear weight                     */
  const uint16_t* bias;    /* bf16 [N] or NULL                                 */
  int64_t M_max;           /* rows X can hold; 0 drops the group               */
  const int64_t* M_dev;    /* device row count (clamped to M_max) or NULL      */
  int32_t K, reserved;
  const int64_t* row_dst;  /* int64 [M_max]: (rank << 40) | row; NULL = row m of out_bases[0] */
} mux_proj_group;

/* Every group's projector + scatter in ONE persistent launch (tiles of group
 * 0, then group 1, ...), sharing N and out_bases.  n_groups <= 2. */
int mux_proj_scatter_grouped(const mux_proj_group* groups, int32_t n_groups, int32_t N,
                             void* const* out_bases, int32_t num_sms, void* stream);

/* Same, and the launch's last CTA then publishes the next epoch to every
 * peer (mux_signal fused into the GEMM: every row store, local or NVLink,
 * is fenced at system scope before the flag).  sync: a zeroed uint32 the
 * kernel re-arms.  e_flags_peers / e_epoch_ctr (optional, NULL = none): a
 * second channel signalled at kernel START without a fence — the
 * "receive windows consumed" permission (mux_signal_ex with fence 0) fused
 * into the launch.  poison (nullable): as for mux_segcopy_ex — a poisoned
 * launch computes nothing and publishes its epoch with MUX_POISON_BIT. */
int mux_proj_scatter_grouped_signal(const mux_proj_group* groups, int32_t n_groups, int32_t N,
                                    void* const* out_bases, int32_t num_sms, int32_t me,
                                    int32_t world, uint64_t* const* flags_peers, uint32_t* sync,
                                    uint64_t* epoch_ctr, uint64_t* const* e_flags_peers,
                                    uint64_t* e_epoch_ctr, const int32_t* poison, void* stream);

/* Decentralized step metadata ("metadata all-gather";
 * SPEC.md:400-402): every rank packs its loader's share of the step (carried
 * sequences and drawn chunks, contiguous ranges in rank order) into a record
 * of mux_meta_record_words(cap_rows, cap_chunks) int32 words:
 *   [n_carry_rows, n_carry_seqs, n_chunk_rows, n_chunks], ids int64[cap_rows],
 *   lens int32[cap_rows], mods int32[cap_rows], carry seq (local) int32[cap_rows],
 *   chunk sizes int32[cap_chunks]   (rows: carry rows first, then chunk rows).
 * After an all-gather of the records (world of them, rank order),
 * mux_assemble_table writes the global step-table blob (ids int64[S] | lens |
 * mods | carry_seq | chunk_off, the layout mux_plan_step reads) in the order
 * the centralized generate_batch produces (workload.py:281-305).  *err
 * (device int32, zero on entry) is set to 1 if a record is malformed or
 * out_words is too small. */
int64_t mux_meta_record_words(int32_t cap_rows, int32_t cap_chunks);
int mux_assemble_table(const int32_t* records, int32_t world, int32_t cap_rows, int32_t cap_chunks,
                       int64_t* out_blob, int64_t out_words, int32_t* err, void* stream);

/* Backward of the projector (no reference kernel; the gradient path of
 * SPEC.md:411 and PAPER.md:1114), on the encoder rank after the gradient
 * return: G bf16 [M_max, N] = dL/dY of the encoder rows in encoder order,
 * X bf16 [M_max, K] = the projector input, W bf16 [N, K] the weight.
 *   dX bf16 [M_max, K] = G . W        (rows < M written)
 *   dW bf16 [N, K]     = G^T . X      (fp32 accumulation, deterministic)
 *   db bf16 [N]        = sum_m G[m,:] (one pass over G, deterministic; NULL = skip)
 * M = *M_dev clamped to M_max (M_dev NULL: M_max).  dX, dW or db may be NULL to
 * skip that product.  Rows [M, round_up(M, 64)) of G and X are zeroed.
 * tcgen05 CTA-pair GEMMs (MN-major operands for dW); K % 256 == 0,
 * N % 256 == 0.  workspace >= mux_proj_backward_workspace(K, N, num_sms)
 * bytes (W^T, split-K partials; one call at a time per workspace — it is
 * stream-ordered scratch); num_sms = SMs the launches may use (0: all). */
size_t mux_proj_backward_workspace(int32_t K, int32_t N, int32_t num_sms);
int mux_proj_backward(const uint16_t* G, const uint16_t* X, const uint16_t* W, int64_t M_max,
                      const int64_t* M_dev, int32_t K, int32_t N, uint16_t* dX, uint16_t* dW,
                      uint16_t* db, void* workspace, size_t workspace_bytes, int32_t num_sms,
                      void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MUX_B200_H */
