"""Data-plane parity on one GPU: pack, stand-in encoder, return + scatter,
bit-exact against the fake-world oracle (oracle/dataplane.py)."""

import numpy as np
import pytest
import torch

from oracle import dataplane as odp
from oracle import planner as oplan
from paper_2605_08962_b200 import configs, planner
from paper_2605_08962_b200.dataplane import MuxPath
from tests.helpers import golden_steps, random_table
from tests.test_gpu_planner import to_table

pytestmark = pytest.mark.gpu


def payload(rows, width, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(rows, width, generator=g).to(torch.bfloat16)


def run_step(t, cap, gbs, d_in, d_llm, method="lpt", check_enc=True):
    o = oplan.plan_step(t, cap, gbs, 1, 1, 1, 1, method)
    arenas_cpu = [payload(int(o["arena_rows"][0, g]), d_in[g], 100 + g) for g in range(2)]
    path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_llm=d_llm, method=method,
                   max_rows=max(int(o["recv_rows"].max()), 1) + 16)
    table = to_table(t)
    dtab = planner.DeviceTable(table, "cuda")
    plan = path.plan(dtab)
    plan.check(table)
    arenas = [a.cuda() for a in arenas_cpu]
    path.llm_view().zero_()
    path.dispatch(plan, arenas)
    path.encode_standin(plan, dtab)
    path.return_scatter(plan)
    torch.cuda.synchronize()
    ar = [[a.view(torch.int16).numpy().view(np.uint16) for a in arenas_cpu]]
    recv, enc_out, llm = odp.run_world(o, t, 1, ar, d_in, (d_llm, d_llm), d_llm)
    for g in range(2):
        n = int(o["recv_rows"][0, g])
        got = path.recv_view(g, n).cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, recv[0][g]), f"recv group {g}"
        if check_enc:
            got = path.enc_view(g, n).cpu().view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(got, enc_out[0][g]), f"encoder stand-in group {g}"
    n = int(o["llm_rows"][0])
    got = path.llm_view(n).cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, llm[0]), "packed LLM input"
    # gradient path: dY at the placeholder rows back to encoder order
    dy = payload(max(n, 1), d_llm, 7).cuda()
    path.grad_return(plan, dy)
    torch.cuda.synchronize()
    want = odp.run_grad(o, 1, [dy.cpu().view(torch.int16).numpy().view(np.uint16)], d_llm)
    for g in range(2):
        r = int(o["recv_rows"][0, g])
        got = path.grad_view(g, r).cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, want[0][g]), f"gradient return group {g}"
    return o


def test_dataplane_golden_steps_narrow(cuda_device):
    """Every golden world-1 step at full token counts, narrow rows (width-agnostic kernels)."""
    n = 0
    for name, st, t, _ in golden_steps():
        if st["world"] != 1:
            continue
        run_step(t, configs.CAPACITY, st["gbs"], (20, 8), 64)
        n += 1
    assert n >= 6


def test_dataplane_sm_return_path(cuda_device):
    """At one GPU the return and gradient copies default to the TMA engine
    (segcopy.cu MUX_COPY_BULK); the SM copy they replaced must still give the
    same bits: the golden-step and full-width cases again with MUX_COPY_BULK=0
    (read once per process, hence the subprocess)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MUX_COPY_BULK="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        f"{__file__}::test_dataplane_golden_steps_narrow",
                        f"{__file__}::test_dataplane_target1_full_width"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_dataplane_target1_full_width(cuda_device):
    """target-1 step 0 at the real widths: 588/512-wide loader rows, 4096-wide returns."""
    for name, st, t, _ in golden_steps():
        if name == "target1" and st["world"] == 1 and st["step"] == 0:
            o = run_step(t, configs.CAPACITY, st["gbs"], (588, 512), 4096, check_enc=False)
            assert int(o["recv_rows"].sum()) > 30000
            return
    raise AssertionError("target1 golden step missing")


def test_dataplane_random_tables(cuda_device):
    rs = np.random.RandomState(21)
    for it in range(25):
        t, cap = random_table(rs)
        try:
            run_step(t, cap, 2, (12, 4), 16, method="kk" if it % 2 else "lpt")
        except ValueError:
            continue


def test_standin_matches_oracle(cuda_device):
    """E(id, t, c) bit patterns for large ids (high 32 bits set)."""
    t = dict(lens=np.array([7, 3, 5]), mods=np.array([1, 3, 2]),
             ids=np.array([2 ** 40 + 5, 99_000_017, 3]), carry_seq=np.zeros(0, np.int64),
             n_carry_seqs=0, chunk_off=[0, 3])
    run_step(t, 16, 1, (8, 8), 24)


@pytest.mark.parametrize("eta", [0, 3000])
def test_dataplane_lssp_one_gpu(cuda_device, eta):
    """LSSP on one GPU (group of 1): DP rows first, then the SP samples, each
    buffer bit-exact against oracle/lssp.py; the packed LLM input is unchanged."""
    from oracle import lssp as olssp
    for name, st, t, _ in golden_steps():
        if name != "target1" or st["world"] != 1 or st["step"] != 1:
            continue
        cap, gbs, d_in, d_llm = configs.CAPACITY, st["gbs"], (20, 8), 64
        o = oplan.plan_step(t, cap, gbs, 1, 1, 1, 1, "lpt")
        lay = olssp.layout(o, t["lens"], 1, eta, 1)
        assert (lay["state"] == 1).any() and (eta == 0 or (lay["state"] == 0).any())
        arenas_cpu = [payload(int(o["arena_rows"][0, g]), d_in[g], 100 + g) for g in range(2)]
        path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_llm=d_llm, method="lpt",
                       lssp_eta=eta, lssp_sp=1)
        table = to_table(t)
        dtab = planner.DeviceTable(table, "cuda")
        plan = path.plan(dtab)
        plan.check(table)
        path.llm_view().zero_()
        path.dispatch(plan, [a.cuda() for a in arenas_cpu])
        path.encode_standin(plan, dtab)
        path.return_scatter(plan)
        torch.cuda.synchronize()
        ar = [[a.view(torch.int16).numpy().view(np.uint16) for a in arenas_cpu]]
        recv, enc_out, llm = olssp.run_world(o, lay, t, 1, ar, d_in, (d_llm, d_llm), d_llm)
        for g in range(2):
            n = int(lay["recv_rows"][0, g])
            got = path.recv_view(g, n).cpu().view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(got, recv[0][g]), f"recv group {g}"
            got = path.enc_view(g, n).cpu().view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(got, enc_out[0][g]), f"encoder rows group {g}"
        n = int(o["llm_rows"][0])
        got = path.llm_view(n).cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, llm[0])
        _, _, llm_plain = odp.run_world(o, t, 1, ar, d_in, (d_llm, d_llm), d_llm)
        assert np.array_equal(got, llm_plain[0]), "LLM input must not depend on the split"
        dy = payload(max(n, 1), d_llm, 7).cuda()
        path.grad_return(plan, dy)
        torch.cuda.synchronize()
        want = olssp.run_grad(lay, 1, [dy.cpu().view(torch.int16).numpy().view(np.uint16)], d_llm)
        for g in range(2):
            r = int(lay["recv_rows"][0, g])
            got = path.grad_view(g, r).cpu().view(torch.int16).numpy().view(np.uint16)
            assert np.array_equal(got, want[0][g]), f"gradient group {g}"
        return
    raise AssertionError("target1 golden step missing")


def test_dataplane_with_text_rows(cuda_device):
    """The whole packed LLM input of a step: modality rows from the return path,
    text rows gathered from a bf16 embedding table by token id."""
    for name, st, t, _ in golden_steps():
        if name != "cfg2" or st["world"] != 1 or st["step"] != 0:
            continue
        cap, gbs, d_in, d_llm = configs.CAPACITY, st["gbs"], (20, 8), 64
        o = oplan.plan_step(t, cap, gbs, 1, 1, 1, 1, "lpt")
        assert o["text_pieces"]
        arenas_cpu = [payload(int(o["arena_rows"][0, g]), d_in[g], 100 + g) for g in range(2)]
        path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_llm=d_llm, method="lpt",
                       text_embed=True)
        table = to_table(t)
        dtab = planner.DeviceTable(table, "cuda")
        plan = path.plan(dtab)
        plan.check(table)
        vocab = 5000
        emb = payload(vocab, d_llm, 11)
        n_text = int(sum(int(L) for L, m in zip(t["lens"], t["mods"]) if m == 0))
        tokens = torch.randint(0, vocab, (max(n_text, 1),), generator=torch.Generator()
                               .manual_seed(4), dtype=torch.int32)
        path.llm_view().zero_()
        path.dispatch(plan, [a.cuda() for a in arenas_cpu])
        path.encode_standin(plan, dtab)
        path.return_scatter(plan)
        path.embed_text(plan, tokens.cuda(), emb.cuda())
        torch.cuda.synchronize()
        path.check_text()
        ar = [[a.view(torch.int16).numpy().view(np.uint16) for a in arenas_cpu]]
        _, _, llm = odp.run_world(o, t, 1, ar, d_in, (d_llm, d_llm), d_llm)
        llm = odp.run_text(o, t, 1, tokens.numpy(), emb.view(torch.int16).numpy().view(np.uint16),
                           llm)
        n = int(o["llm_rows"][0])
        got = path.llm_view(n).cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, llm[0])
        # every LLM row is written: modality + text rows fill the packed buffer
        assert int(plan.header()[_lib_H_TEXT_ROWS()]) + int(o["recv_rows"].sum()) == n
        bad = tokens.clone()
        bad[0] = vocab
        path.embed_text(plan, bad.cuda(), emb.cuda())
        with pytest.raises(ValueError, match="outside"):
            path.check_text()
        return
    raise AssertionError("cfg2 golden step missing")


def _lib_H_TEXT_ROWS():
    from paper_2605_08962_b200 import _lib
    return _lib.H_TEXT_ROWS


def test_all_text_step_moves_no_modality_rows(cuda_device):
    """A step with text samples only: no dispatch, no return, the projector GEMM
    sees M = 0 on the device; the text rows are still gathered."""
    lens = np.array([4000, 3000, 9000, 120, 0, 5000])
    t = dict(lens=lens, mods=np.zeros(len(lens), np.int64), ids=np.arange(10, 10 + len(lens)),
             carry_seq=np.zeros(0, np.int64), n_carry_seqs=0, chunk_off=[0, len(lens)])
    o = oplan.plan_step(t, configs.CAPACITY, 1, 1, 1, 1, 1, "lpt")
    assert int(o["recv_rows"].sum()) == 0 and not o["pieces"]
    path = MuxPath(capacity=configs.CAPACITY, gbs=1, dp=1, d_in=(20, 8), d_enc=(256, 256),
                   d_llm=256, projector=True, text_embed=True)
    for g in range(2):
        path.set_projector(g, torch.randn(256, 256, device="cuda").to(torch.bfloat16))
    table = to_table(t)
    dtab = planner.DeviceTable(table, "cuda")
    plan = path.plan(dtab)
    h = plan.check(table)
    assert int(h[3]) == 0 and int(h[4]) == 0  # no dispatch segments, no return pieces
    path.llm_view().zero_()
    path.dispatch(plan, [torch.zeros(1, 20, dtype=torch.bfloat16, device="cuda"),
                         torch.zeros(1, 8, dtype=torch.bfloat16, device="cuda")])
    path.return_scatter(plan)
    emb = payload(100, 256, 3)
    tokens = torch.randint(0, 100, (int(lens.sum()),), dtype=torch.int32)
    path.embed_text(plan, tokens.cuda(), emb.cuda())
    torch.cuda.synchronize()
    path.check_text()
    n = int(o["llm_rows"][0])
    llm = [np.zeros((n, 256), np.uint16)]
    llm = odp.run_text(o, t, 1, tokens.numpy(), emb.view(torch.int16).numpy().view(np.uint16),
                       llm)
    got = path.llm_view(n).cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, llm[0])


@pytest.mark.parametrize("overlap", [False, True])
def test_streaming_pipeline_matches_list_form(cuda_device, overlap):
    """run_pipeline(n=, prepare=): every step uploaded from pinned host memory
    into one of two reused device slots on a copy stream (the bench's e2e form),
    slots released through path.step_done; recv windows and LLM rows of every
    step equal the list form's, also across two calls issued without a sync."""
    from paper_2605_08962_b200.dataplane import MuxPath
    steps = [(st, t) for nm, st, t, _ in golden_steps() if nm == "target1" and st["world"] == 1]
    steps = (steps * 2)[:6]
    cap, gbs = configs.CAPACITY, steps[0][0]["gbs"]
    d_in, d_llm = (20, 8), 64
    tables = [to_table(t) for _, t in steps]
    os_ = [oplan.plan_step(t, cap, gbs, 1, 1, 1, 1, "lpt") for _, t in steps]
    host_ar = [[payload(max(int(o["arena_rows"][0, g]), 1), d_in[g], 300 + 7 * k + g)
                .pin_memory() for g in range(2)] for k, o in enumerate(os_)]

    def run(stream_form, calls):
        path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_llm=d_llm,
                       overlap_dispatch=overlap)
        recv, llm = [], []

        def encoder(k, p, s):
            o = os_[len(recv)]
            recv.append([path.recv_view(g, int(o["recv_rows"][0, g])).clone() for g in range(2)])
            path.llm_view().zero_()  # text rows stay zero, as in the oracle
            path.encode_standin(p, dtab_of[len(recv) - 1], s)

        def after(k, p, s):
            llm.append(path.llm_view(int(os_[len(llm)]["llm_rows"][0])).clone())

        dtab_of = {}
        if not stream_form:
            tabs = [planner.DeviceTable(t, "cuda") for t in tables]
            for k, d in enumerate(tabs):
                dtab_of[k] = d
            path.run_pipeline([(tabs[k], [a.cuda() for a in host_ar[k]]) for k in range(6)],
                              encoder=encoder, after_step=after)
        else:
            up = torch.cuda.Stream()
            blobs = [torch.from_numpy(t.blob()).pin_memory() for t in tables]
            slot_tab = [torch.empty(max(b.numel() for b in blobs), dtype=torch.int64,
                                    device="cuda") for _ in range(2)]
            slot_ar = [[torch.empty(max(h[g].numel() for h in host_ar), dtype=torch.bfloat16,
                                    device="cuda") for g in range(2)] for _ in range(2)]
            freed = [None, None]
            base = [0]

            def prepare(k):
                j = base[0] + k
                slot = j % 2
                if freed[slot] is not None:
                    up.wait_event(freed[slot])
                with torch.cuda.stream(up):
                    b = slot_tab[slot][:blobs[j].numel()]
                    b.copy_(blobs[j], non_blocking=True)
                    ars = []
                    for g in range(2):
                        h = host_ar[j][g]
                        a = slot_ar[slot][g][:h.numel()].view(h.shape)
                        a.copy_(h, non_blocking=True)
                        ars.append(a)
                ev = torch.cuda.Event()
                ev.record(up)
                dtab_of[j] = planner.DeviceTable.from_blob(tables[j], b)
                return dtab_of[j], ars, ev

            def after_s(k, p, s):
                after(k, p, s)
                if path.step_done is not None:
                    s.wait_event(path.step_done)
                e = torch.cuda.Event()
                e.record(s)
                freed[(base[0] + k) % 2] = e

            per = 6 // calls
            for c in range(calls):  # no synchronisation between the calls
                base[0] = c * per
                path.run_pipeline(n=per, prepare=prepare, encoder=encoder, after_step=after_s)
        torch.cuda.synchronize()
        return recv, llm

    want_recv, want_llm = run(False, 1)
    for k, ((st, t), o) in enumerate(zip(steps, os_)):  # the list form against the oracle
        ar = [[a.view(torch.int16).numpy().view(np.uint16) for a in host_ar[k]]]
        recv, _, llm = odp.run_world(o, t, 1, ar, d_in, (d_llm, d_llm), d_llm)
        for g in range(2):
            assert np.array_equal(want_recv[k][g].cpu().view(torch.int16).numpy()
                                  .view(np.uint16), recv[0][g]), (k, g)
        assert np.array_equal(want_llm[k].cpu().view(torch.int16).numpy().view(np.uint16),
                              llm[0]), k
    for calls in (1, 2):
        got_recv, got_llm = run(True, calls)
        for k in range(6):
            for g in range(2):
                assert torch.equal(got_recv[k][g], want_recv[k][g]), (calls, k, g)
            assert torch.equal(got_llm[k], want_llm[k]), (calls, k)


def test_dispatch_reads_pinned_host_rows(cuda_device):
    """The fused loader transfer (bench e2e `fused_loader`): the
    dispatch kernel reads each sample's rows straight from pinned host memory
    (UVA) into the receive windows — bit-exact against the oracle."""
    from paper_2605_08962_b200.dataplane import MuxPath
    for name, st, t, _ in golden_steps():
        if name == "target1" and st["world"] == 1 and st["step"] == 1:
            break
    cap, gbs, d_in = configs.CAPACITY, st["gbs"], (588, 512)
    o = oplan.plan_step(t, cap, gbs, 1, 1, 1, 1, "lpt")
    host = [payload(max(int(o["arena_rows"][0, g]), 1), d_in[g], 40 + g).pin_memory()
            for g in range(2)]
    path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_llm=64)
    table = to_table(t)
    plan = path.plan(planner.DeviceTable(table, "cuda"))
    plan.check(table)
    path.dispatch(plan, host)
    torch.cuda.synchronize()
    ar = [[a.view(torch.int16).numpy().view(np.uint16) for a in host]]
    recv, _, _ = odp.run_world(o, t, 1, ar, d_in, (64, 64), 64)
    for g in range(2):
        n = int(o["recv_rows"][0, g])
        got = path.recv_view(g, n).cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, recv[0][g]), g
