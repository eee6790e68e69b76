"""One small pass over every kernel of libmuxb200.so at one GPU, for
compute-sanitizer (memcheck / racecheck / synccheck; one tool per run):

  compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py

planner (step plan with LSSP, CpHybrid, text segments; pack mode), segment copies
(dispatch, return, gradient), encoder stand-in, text rows, row maps, projector
GEMM forward (pair and single-CTA) and backward, metadata assembly, flag
signal/wait.  Shapes are small so the tools finish in minutes."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import planner as oplan  # noqa: E402
from oracle import workload as owork  # noqa: E402
from paper_2605_08962_b200 import _lib, configs, planner  # noqa: E402
from paper_2605_08962_b200.dataplane import MuxPath  # noqa: E402


def main():
    torch.cuda.set_device(0)
    cfg = configs.CONFIGS["target1"]
    descs = owork.descs_from_config(configs.DATASETS, cfg["datasets"])
    cap, gbs = 2048, 2
    for d in descs.values():
        d["max_len"] = cap
    _, _, drawn, chunks = owork.generate(descs, cfg["phases"], False, 0, cfg["seed"], gbs, 1, 1,
                                         cap)
    t = oplan.step_table([], drawn, chunks, {})
    table = planner.StepTable(t["lens"].astype(np.int32), t["mods"].astype(np.int32), t["ids"],
                              t["carry_seq"].astype(np.int32), 0,
                              np.asarray(t["chunk_off"], np.int32))
    d_in, d_llm = (24, 16), 64
    o = oplan.plan_step(t, cap, gbs, 1, 1, 1)
    arenas = [torch.randn(max(int(o["arena_rows"][0, g]), 1), d_in[g], device="cuda")
              .to(torch.bfloat16) for g in range(2)]
    for kw in ({}, {"text_embed": True}, {"lssp_eta": 256, "lssp_sp": 1}):
        path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_llm=d_llm, **kw)
        dtab = planner.DeviceTable(table, "cuda")
        plan = path.plan(dtab)
        plan.check(table)
        path.dispatch(plan, arenas)
        path.encode_standin(plan, dtab)
        path.return_scatter(plan)
        dy = torch.randn(path.max_llm_rows, d_llm, device="cuda").to(torch.bfloat16)
        path.grad_return(plan, dy)
        if kw.get("text_embed"):
            tok = torch.randint(0, 100, (int(sum(t["lens"])),), device="cuda", dtype=torch.int32)
            emb = torch.randn(100, d_llm, device="cuda").to(torch.bfloat16)
            path.embed_text(plan, tok, emb)
        torch.cuda.synchronize()
    planner.device_pack([list(range(0))], cap) if False else planner.device_pack([[]], cap)
    # projector forward (pair + single CTA) and backward
    d_enc = (256, 256)
    for pair in ("1", "0"):
        os.environ["MUX_GEMM_2CTA"] = pair
        path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_enc=d_enc, d_llm=256,
                       projector=True)
        for g in range(2):
            path.set_projector(g, torch.randn(256, 256, device="cuda").to(torch.bfloat16),
                               torch.randn(256, device="cuda").to(torch.bfloat16))
        dtab = planner.DeviceTable(table, "cuda")
        plan = path.plan(dtab)
        path.dispatch(plan, arenas)
        path.encode_standin(plan, dtab)
        path.return_scatter(plan)
        torch.cuda.synchronize()
        break  # the library reads MUX_GEMM_2CTA once per process
    dy = torch.randn(path.max_llm_rows, 256, device="cuda").to(torch.bfloat16)
    path.grad_return(plan, dy)
    path.projector_backward(0, plan=plan)
    torch.cuda.synchronize()
    # metadata assembly
    recs = np.stack([table.shard(r, 2).record(256, 8) for r in range(2)])
    dev = torch.from_numpy(recs.reshape(-1)).cuda()
    blob = torch.empty(table.blob().size, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().mux_assemble_table(dev.data_ptr(), 2, 256, 8, blob.data_ptr(),
                                             blob.numel(), err.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream))
    # flags: signal then wait on one's own slot (world 1)
    L = _lib.lib()
    flags = torch.zeros(1, dtype=torch.int64, device="cuda")
    fptrs = torch.tensor([flags.data_ptr()], dtype=torch.int64, device="cuda")
    ep = torch.zeros(1, dtype=torch.int64, device="cuda")
    werr = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.mux_signal(0, 1, fptrs.data_ptr(), ep.data_ptr(), s))
    _lib.check(L.mux_wait(1, flags.data_ptr(), ep.data_ptr(), 1000, werr.data_ptr(), s))
    torch.cuda.synchronize()
    assert int(err.item()) == 0 and int(werr.item()) == 0
    print("sanitize smoke ok", flush=True)


if __name__ == "__main__":
    main()
