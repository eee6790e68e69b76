// Decentralized step metadata (loaders hold their own
// samples; each reordering group starts with "a metadata all-gather operation
// to exchange data size").
//
// Every rank's loader holds a contiguous share of the step: carried sequences
// [q_r, q_r+1) and drawn chunks [c_r, c_r+1) (planner.StepTable.shard).  It
// packs them into a fixed-size record (layout below); one all-gather over
// NVLink (NCCL, torch.distributed) puts every record on every rank, and
// assemble_kernel rebuilds the global step table blob — carry rows of rank
// 0, 1, ... (sequence ids offset by the lower ranks' carried sequences), then
// chunk rows of rank 0, 1, ... with chunk offsets — in exactly the table order
// generate_batch packs (workload.py:281-305), so the device planner yields the
// plan of the centralized table bit for bit.
//
// Record of one rank (int32 words; cap = rows capacity, capc = chunk capacity):
//   [0..3]   n_carry_rows, n_carry_seqs, n_chunk_rows, n_chunks
//   ids      int64[cap]   (words 4 .. 4 + 2 cap)
//   lens     int32[cap]
//   mods     int32[cap]
//   cseq     int32[cap]   local carried-sequence index of every carry row
//   csize    int32[capc]  rows of every drawn chunk
// Output blob (planner.StepTable.blob): ids int64[S] | lens int32[S] |
// mods int32[S] | carry_seq int32[nc] | chunk_off int32[n_chunks + 1].

#include "mux_common.cuh"

namespace mux {

constexpr int kMetaMaxWorld = 32;

__global__ void assemble_kernel(const int32_t* rec, int world, int cap, int capc,
                                int64_t* out, int64_t out_words, int32_t* err) {
  __shared__ int s_cr[kMetaMaxWorld + 1], s_cs[kMetaMaxWorld + 1], s_kr[kMetaMaxWorld + 1],
      s_kn[kMetaMaxWorld + 1];
  const int64_t rec_words = 4 + 2 * (int64_t)cap + 3 * (int64_t)cap + capc;
  if (threadIdx.x == 0) {
    int cr = 0, cs = 0, kr = 0, kn = 0, bad = 0;
    for (int r = 0; r < world; ++r) {
      const int32_t* h = rec + r * rec_words;
      s_cr[r] = cr;
      s_cs[r] = cs;
      s_kr[r] = kr;
      s_kn[r] = kn;
      if (h[0] < 0 || h[2] < 0 || h[0] + h[2] > cap || h[3] < 0 || h[3] > capc || h[1] < 0)
        bad = 1;
      cr += h[0];
      cs += h[1];
      kr += h[2];
      kn += h[3];
    }
    s_cr[world] = cr;
    s_cs[world] = cs;
    s_kr[world] = kr;
    s_kn[world] = kn;
    const int64_t S = cr + kr;
    const int64_t need = S + (2 * S + cr + kn + 1 + 1) / 2;
    if (bad || need > out_words) *err = 1;
  }
  __syncthreads();
  if (*(volatile int32_t*)err) return;
  const int nc = s_cr[world], S = nc + s_kr[world], nch = s_kn[world];
  int64_t* ids = out;
  int32_t* i32 = reinterpret_cast<int32_t*>(out + S);
  int32_t* lens = i32;
  int32_t* mods = i32 + S;
  int32_t* cseq = i32 + 2 * S;
  int32_t* coff = i32 + 2 * S + nc;
  for (int r = 0; r < world; ++r) {
    const int32_t* h = rec + r * rec_words;
    const int64_t* rid = reinterpret_cast<const int64_t*>(h + 4);
    const int32_t* rlen = h + 4 + 2 * cap;
    const int32_t* rmod = rlen + cap;
    const int32_t* rcs = rmod + cap;
    const int32_t* rsz = rcs + cap;
    const int ncr = h[0], nkr = h[2], nk = h[3];
    for (int t = threadIdx.x; t < ncr + nkr; t += blockDim.x) {
      const int dst = t < ncr ? s_cr[r] + t : nc + s_kr[r] + (t - ncr);
      ids[dst] = rid[t];
      lens[dst] = rlen[t];
      mods[dst] = rmod[t];
      if (t < ncr) cseq[dst] = rcs[t] + s_cs[r];
    }
    if (threadIdx.x == 0) {  // chunk offsets of this rank's chunks
      int o = nc + s_kr[r];
      for (int c = 0; c < nk; ++c) {
        coff[s_kn[r] + c] = o;
        o += rsz[c];
      }
      if (r == world - 1) {
        coff[nch] = S;
        if ((2 * S + nc + nch + 1) & 1) coff[nch + 1] = 0;  // pad the last int64 word
      }
    }
  }
}

}  // namespace mux

using namespace mux;

extern "C" int64_t mux_meta_record_words(int32_t cap_rows, int32_t cap_chunks) {
  return 4 + 2 * (int64_t)cap_rows + 3 * (int64_t)cap_rows + cap_chunks;
}

extern "C" int mux_assemble_table(const int32_t* records, int32_t world, int32_t cap_rows,
                                  int32_t cap_chunks, int64_t* out_blob, int64_t out_words,
                                  int32_t* err, void* stream) {
  if (world < 1 || world > kMetaMaxWorld || cap_rows < 0 || cap_chunks < 0 || !records ||
      !out_blob || !err) {
    set_error("mux_assemble_table: need 1 <= world <= %d, capacities >= 0, non-null buffers",
              kMetaMaxWorld);
    return MUX_ERR_VALUE;
  }
  assemble_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      records, world, cap_rows, cap_chunks, out_blob, out_words, err);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
