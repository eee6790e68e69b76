"""Device planner parity: every plan array bit-exact against the CPU oracle."""

import numpy as np
import pytest

from oracle import dataplane as odp
from oracle import planner as oplan
from oracle import workload as owork
from paper_2605_08962_b200 import balance, configs, costs, planner, workload as W
from tests.helpers import golden, golden_steps, oracle_plan, random_table

pytestmark = pytest.mark.gpu


def to_table(t):
    return planner.StepTable(np.asarray(t["lens"], np.int32), np.asarray(t["mods"], np.int32),
                             np.asarray(t["ids"], np.int64), np.asarray(t["carry_seq"], np.int32),
                             int(t["n_carry_seqs"]), np.asarray(t["chunk_off"], np.int32))


def device_plan(t, cap, gbs, dp, sp, world, me, method="lpt", pooled=False, reorder_group=0,
                cost=None):
    table = to_table(t)
    cfg = planner.make_cfg(table, cap, gbs, dp, sp, world, 1, method, pooled, me,
                           row_bytes_in=(1176, 1024), row_bytes_ret=(8192, 8192),
                           reorder_group=reorder_group, cost=cost)
    plan = planner.plan_step(planner.DeviceTable(table, "cuda"), cfg)
    plan.check(table)
    return plan.host()


def assert_plan_equal(d, o, t, me):
    S = len(t["lens"])
    for k in ("seq", "off", "span"):
        assert np.array_equal(d[k][:S], o[k]), k
    assert int(d["header"][2]) == o["n_seq"]
    assert np.array_equal(d["fills"], o["fills"])
    inb = o["in_batch"]
    for k in ("origin", "origin_pos", "enc", "arena_off", "enc_off"):
        assert np.array_equal(d[k][inb], o[k][inb]), k
    g = np.asarray(d["group"])
    assert np.array_equal(g, o["group"])
    assert np.array_equal(d["cu"], o["cu"])
    assert np.array_equal(d["arena_rows"], o["arena_rows"])
    assert np.array_equal(d["recv_rows"], o["recv_rows"])
    assert np.array_equal(d["llm_rows"], o["llm_rows"])
    assert np.array_equal(d["row_base"].reshape(o["row_base"].shape), o["row_base"])
    assert np.array_equal(d["dseg"], odp.dispatch_by_rank(o, t["lens"], me))
    assert np.array_equal(d["rseg"], odp.pieces_by_rank(o, me))
    assert np.array_equal(d["gseg"], odp.grad_by_rank(o, me))


@pytest.mark.parametrize("method", ["lpt", "kk", "lpt_local", "lpt_local_rw"])
def test_plan_matches_oracle_on_golden_steps(cuda_device, method):
    n = 0
    for name, st, t, _ in golden_steps():
        o = oracle_plan(t, st, method)
        world, dp = st["world"], st["dp"]
        for me in range(world):
            d = device_plan(t, configs.CAPACITY, st["gbs"], dp, world // dp, world, me, method)
            assert_plan_equal(d, o, t, me)
            n += 1
    assert n > 20


FLOPS = tuple(costs.encoder_cost_params(costs.ModelSpec(f"enc{g}", costs.ModelKind.ENCODER,
                                                       p, layers, hidden, 16))
              for g, (p, layers, hidden) in enumerate(configs.ENCODER_SHAPES))


@pytest.mark.parametrize("method", ["lpt", "kk", "lpt_local", "lpt_local_rw"])
@pytest.mark.parametrize("reorder_group,cost", [(2, None), (4, None), (0, FLOPS), (2, FLOPS),
                                                (1, None)])
def test_reorder_groups_and_flops_costs_match_oracle(cuda_device, method, reorder_group, cost):
    """Reorder groups of consecutive ranks and the
    flops-weighted cost (costs.py:108-124): every 4- and 8-rank golden step,
    every rank's plan bit-exact; samples stay inside their origin's group."""
    n = 0
    for name, st, t, _ in golden_steps():
        world, dp = st["world"], st["dp"]
        if world < 4 or (reorder_group and world % reorder_group):
            continue
        o = oplan.plan_step(t, configs.CAPACITY, st["gbs"], dp, world // dp, world, 1, method,
                            reorder_group=reorder_group, cost=cost)
        rg = reorder_group or world
        e = o["enc"] >= 0
        assert np.array_equal(o["enc"][e] // rg, o["origin"][e] // rg)
        for me in range(world):
            d = device_plan(t, configs.CAPACITY, st["gbs"], dp, world // dp, world, me, method,
                            reorder_group=reorder_group, cost=cost)
            assert_plan_equal(d, o, t, me)
            n += 1
    assert n >= 8


def test_plan_matches_oracle_random_tables(cuda_device):
    rs = np.random.RandomState(11)
    checked = 0
    for it in range(120):
        t, cap = random_table(rs)
        world, dp = [(1, 1), (2, 2), (2, 1), (4, 4), (4, 2), (8, 8), (8, 2), (8, 1)][it % 8]
        sp = world // dp
        gbs = dp * int(rs.randint(1, 3))
        method = ("kk", "lpt", "lpt_local", "lpt_local_rw")[it % 4]
        pooled = it % 5 == 0
        try:
            o = oplan.plan_step(t, cap, gbs, dp, sp, world, 1, method, pooled)
        except ValueError as e:
            with pytest.raises(ValueError) as ei:
                device_plan(t, cap, gbs, dp, sp, world, 0, method, pooled)
            assert str(ei.value) == str(e)
            continue
        me = int(rs.randint(0, world))
        d = device_plan(t, cap, gbs, dp, sp, world, me, method, pooled)
        assert_plan_equal(d, o, t, me)
        checked += 1
    assert checked > 60


def test_plan_errors_match_reference_messages(cuda_device):
    t = dict(lens=np.array([4, 20, 5, 30]), mods=np.array([1, 1, 1, 1]),
             ids=np.array([3, 7, 1, 9]), carry_seq=np.zeros(0, np.int64), n_carry_seqs=0,
             chunk_off=[0, 4])
    with pytest.raises(W.PackingError, match=r"^sample 7 \(20 tokens\) exceeds capacity 16$"):
        device_plan(t, 16, 2, 1, 1, 1, 0)
    t["lens"] = np.array([4, 2, 5, 3])
    with pytest.raises(W.ConfigError, match="global batch 3 not divisible by dp 2"):
        device_plan(t, 16, 3, 2, 1, 2, 0)
    with pytest.raises(ValueError, match=r"^need 4 sequences, have 1$"):
        device_plan(t, 16, 4, 1, 1, 1, 0)


def test_hybrid_pack_matches_reference_golden(cuda_device):
    P = golden("pack_cases.json")
    chunks = []
    for c in P["cases"]:
        samples = [W.Sample(i, W.Modality.IMAGE, "x", L) for i, L in zip(c["ids"], c["lens"])]
        got = W.hybrid_pack(samples, c["cap"])
        assert [[list(sp) for sp in q.spans] for q in got] == c["seqs"]
        if c["cap"] == 1000:
            chunks.append((samples, c["seqs"]))
    # several chunks in one launch (one CTA per chunk)
    res = planner.device_pack([s for s, _ in chunks], 1000)
    for (s, want), got in zip(chunks, res):
        assert [[list(sp) for sp in q.spans] for q in got] == want
    for e in P["errors"]:
        samples = [W.Sample(i, W.Modality.AUDIO, "x", L) for i, L in zip(e["ids"], e["lens"])]
        with pytest.raises(W.PackingError) as ei:
            W.hybrid_pack(samples, e["cap"])
        assert str(ei.value) == e["message"]


def test_generate_batch_matches_reference_golden(cuda_device):
    G = golden("configs.json")
    for name in ("cfg2", "cfg4", "target1", "cfg5"):
        cfg = configs.CONFIGS[name]
        reg, sched = configs.build(W, name)
        recs = [s for s in G[name]["steps"] if s["world"] == (8 if name in ("cfg4", "cfg5") else 1)]
        carry = None
        for st in recs:
            drawn = []
            b, carry = W.generate_batch(reg, sched, st["step"], cfg["seed"], st["gbs"], st["dp"], 1,
                                        configs.CAPACITY, carry if cfg["carry"] else None, drawn)
            assert [[list(sp) for sp in q.spans] for q in b.sequences] == st["batch"]
            assert [[list(sp) for sp in q.spans] for q in carry] == st["carry_out"]
            assert [[s.id, s.modality.value, s.dataset, s.length] for s in drawn] == st["drawn"]


@pytest.mark.parametrize("method", ["lpt", "kk"])
def test_partition_matches_oracle(cuda_device, method):
    rs = np.random.RandomState(5)
    for _ in range(40):
        g = int(rs.choice([1, 2, 3, 4, 8]))
        w = rs.lognormal(7, 1.0, size=int(rs.randint(1, 300))).round().tolist()
        ids = rs.permutation(len(w)).tolist()
        if method == "kk":
            want = oplan.kk_assign([float(x) for x in w], g) if g > 1 else [0] * len(w)
            got = balance.kk_partition(w, g)
        else:
            want = oplan.lpt_assign([float(x) for x in w], ids, g)
            got = balance.lpt_partition(w, g, ids=ids)
        assert list(got) == list(want)
    assert list(balance.kk_partition([8, 7, 6, 5, 4], 2)) == [1, 0, 1, 0, 0]


def test_plan_reshard_matches_oracle(cuda_device):
    from paper_2605_08962_b200 import reshard
    from paper_2605_08962_b200 import costs
    for name, st, t, _ in golden_steps():
        if st["world"] != 1:
            continue
        seqs = [W.PackedSequence(configs.CAPACITY, [tuple(x) for x in q]) for q in st["batch"]]
        raw = [[tuple(x) for x in q] for q in st["batch"]]
        for sp in (2, 4, 8):
            got = reshard.plan_reshard(seqs, sp, "ulysses")
            want, loads = oplan.plan_reshard(raw, sp, "ulysses")
            assert got.shard_map == want and got.tokens_per_rank == loads
        for cp, thr in ((2, None), (4, 4096), (4, 1024)):
            got = reshard.plan_reshard(seqs, cp, "cp_hybrid", cp_threshold=thr)
            want, loads = oplan.plan_reshard(raw, cp, "cp_hybrid", cp_threshold=thr,
                                             capacity=configs.CAPACITY)
            assert got.shard_map == want and got.tokens_per_rank == loads
            ev, sec = reshard.dispatch_cost(got, costs.CommModel())
            assert sec > 0 and len(ev) == len(seqs)
    assert reshard.dispatch_cost(reshard.ReshardPlan("ulysses"), costs.CommModel()) == ([], 0.0)


def test_grouped_reorder_and_restore(cuda_device):
    # [10,1,1,1] over 4 ranks -> max stays 10, imbalance 10/3.25;
    # reorder then restore == original order, for KK and LPT
    for method in ("kk", "lpt"):
        g = balance.ReorderGroup([0, 1, 2, 3], [[W.Sample(i, W.Modality.IMAGE, "x", L)]
                                                for i, L in enumerate([10, 1, 1, 1])])
        out, rec = balance.grouped_reorder(g, 1, method)
        loads = [sum(s.length for s in lst) for lst in out]
        assert max(loads) == 10 and balance.imbalance(loads) == 10 / 3.25
        back = balance.restore_order(rec, out)
        assert [[s.id for s in lst] for lst in back] == [[0], [1], [2], [3]]
    rs = np.random.RandomState(4)
    lists = [[W.Sample(100 * r + j, W.Modality.AUDIO, "x", int(rs.randint(1, 5000)))
              for j in range(int(rs.randint(0, 9)))] for r in range(4)]
    lists[0] += [W.Sample(999 + j, W.Modality.VIDEO, "x", 16000) for j in range(4)]  # skewed rank
    pre = [sum(s.length for s in lst) for lst in lists]
    before = [[(s.origin_rank, s.origin_pos) for s in lst] for lst in lists]
    out, rec = balance.grouped_reorder(balance.ReorderGroup([0, 1, 2, 3], lists), 2, "kk")
    # the caller's Samples are not mutated (reference ops return new objects)
    assert [[(s.origin_rank, s.origin_pos) for s in lst] for lst in lists] == before
    assert all(s.origin_rank >= 0 for lst in out for s in lst)
    post = [sum(s.length for s in lst) for lst in out]
    assert balance.imbalance(post) < balance.imbalance(pre)
    back = balance.restore_order(rec, out)
    assert [[s.id for s in lst] for lst in back] == [[s.id for s in lst] for lst in lists]
    with pytest.raises(ValueError):
        bad = balance.ReorderRecord(forward={(0, 0): (0, 0), (0, 1): (0, 0)}, shape=[2])
        balance.restore_order(bad, [[1, 2]])
    assert balance.zero_redundancy_filter(None, 1, 4, 16) == [1, 5, 9, 13]


def lssp_device_plan(t, cap, gbs, dp, sp, world, me, method, sp_enc, eta, reorder_group=0):
    table = to_table(t)
    cfg = planner.make_cfg(table, cap, gbs, dp, sp, world, 1, method, False, me,
                           row_bytes_in=(1176, 1024), row_bytes_ret=(8192, 8192),
                           lssp_sp=sp_enc, lssp_eta=eta, reorder_group=reorder_group)
    plan = planner.plan_step(planner.DeviceTable(table, "cuda"), cfg)
    plan.check(table)
    return plan.host()


def assert_lssp_equal(d, o, lay, t, me):
    from oracle import lssp as olssp
    items = np.flatnonzero(o["enc"] >= 0)
    assert np.array_equal(d["lssp_state"][items], lay["state"][items])
    for i in items:
        cols = 1 if lay["state"][i] == 0 else lay["sp_enc"]
        assert np.array_equal(d["lssp_row"][i, :cols], lay["row"][i, :cols]), i
    assert np.array_equal(d["recv_rows"], lay["recv_rows"])
    assert np.array_equal(d["dseg"], olssp.dispatch_by_rank(o, lay, t["lens"], me))
    assert np.array_equal(d["rseg"], olssp.return_by_rank(lay, me))
    assert np.array_equal(d["gseg"], olssp.grad_by_rank(lay, me))
    h = d["header"]
    assert [int(h[12]), int(h[13])] == lay["recv_rows"][me].tolist()


@pytest.mark.parametrize("sp_enc", [1, 2, 4, 8])
def test_lssp_plan_matches_oracle_on_golden_steps(cuda_device, sp_enc):
    from oracle import lssp as olssp
    n = 0
    for name, st, t, _ in golden_steps():
        world, dp = st["world"], st["dp"]
        if world % sp_enc:
            continue
        o = oracle_plan(t, st, "lpt_local")
        lens = np.asarray(t["lens"])
        items = np.flatnonzero(o["enc"] >= 0)
        for eta in (0, int(np.median(lens[items])) if len(items) else 0, 4096):
            lay = olssp.layout(o, lens, world, eta, sp_enc)
            for me in range(world):
                d = lssp_device_plan(t, configs.CAPACITY, st["gbs"], dp, world // dp, world, me,
                                     "lpt_local", sp_enc, eta)
                assert_lssp_equal(d, o, lay, t, me)
                n += 1
    assert n > 10


def test_lssp_plan_matches_oracle_random_tables(cuda_device):
    from oracle import lssp as olssp
    rs = np.random.RandomState(17)
    checked = 0
    for it in range(80):
        t, cap = random_table(rs)
        world, dp = [(2, 2), (4, 4), (4, 2), (8, 8), (8, 4), (2, 1)][it % 6]
        sp_enc = int(rs.choice([g for g in (1, 2, 4, 8) if world % g == 0]))
        sp = world // dp
        gbs = dp * int(rs.randint(1, 3))
        try:
            o = oplan.plan_step(t, cap, gbs, dp, sp, world, 1, "lpt")
        except ValueError:
            continue
        eta = int(rs.randint(0, cap + 1))
        lay = olssp.layout(o, t["lens"], world, eta, sp_enc)
        me = int(rs.randint(0, world))
        d = lssp_device_plan(t, cap, gbs, dp, sp, world, me, "lpt", sp_enc, eta)
        assert_lssp_equal(d, o, lay, t, me)
        checked += 1
    assert checked > 40


def test_lssp_rejects_bad_groups(cuda_device):
    t = golden_steps().__next__()[2]
    table = to_table(t)
    for sp_enc in (3, 9):
        cfg = planner.make_cfg(table, configs.CAPACITY, 4, 4, 1, 4, 1, "lpt", False, 0,
                               lssp_sp=sp_enc, lssp_eta=10)
        with pytest.raises(ValueError, match="LSSP"):
            planner.plan_step(planner.DeviceTable(table, "cuda"), cfg)


def cp_device_plan(t, cap, gbs, dp, sp, world, me, method, thr, lssp_sp=0, eta=0,
                   reorder_group=0, cost=None):
    table = to_table(t)
    cfg = planner.make_cfg(table, cap, gbs, dp, sp, world, 1, method, False, me,
                           row_bytes_in=(1176, 1024), row_bytes_ret=(8192, 8192),
                           reshard="cp_hybrid", cp_threshold=thr or 0,
                           lssp_sp=lssp_sp, lssp_eta=eta, reorder_group=reorder_group,
                           cost=cost)
    plan = planner.plan_step(planner.DeviceTable(table, "cuda"), cfg)
    plan.check(table)
    return plan.host()


def assert_cp_equal(d, c, t, me):
    gb = c["shard_len"].size
    assert np.array_equal(d["shard_len"][:gb], c["shard_len"].reshape(-1))
    assert np.array_equal(d["row_base"][:gb], c["row_base"].reshape(-1))
    assert np.array_equal(d["llm_rows"], c["llm_rows"])
    assert np.array_equal(d["recv_rows"], c["recv_rows"])
    assert np.array_equal(d["dseg"], odp.dispatch_by_rank(c, t["lens"], me))
    assert np.array_equal(d["rseg"], odp.pieces_by_rank(c, me))
    assert np.array_equal(d["gseg"], odp.grad_by_rank(c, me))


@pytest.mark.parametrize("thr", [None, 1024, 1])
def test_cp_hybrid_plan_matches_oracle(cuda_device, thr):
    from oracle import cphybrid as ocph
    n = 0
    for name, st, t, _ in golden_steps():
        for world, dp in ((2, 1), (4, 1), (4, 2), (8, 2), (8, 1)):
            sp = world // dp
            gbs = st["gbs"] * dp // st["dp"] if st["gbs"] % st["dp"] == 0 else st["gbs"]
            try:
                o = oplan.plan_step(t, configs.CAPACITY, gbs, dp, sp, world, 1, "lpt")
            except ValueError:
                continue
            c = ocph.place(o, t, gbs, dp, sp, configs.CAPACITY, thr)
            for me in range(world):
                d = cp_device_plan(t, configs.CAPACITY, gbs, dp, sp, world, me, "lpt", thr)
                assert_cp_equal(d, c, t, me)
                n += 1
    assert n > 20


def test_cp_hybrid_with_lssp_matches_oracle(cuda_device):
    from oracle import cphybrid as ocph
    from oracle import lssp as olssp
    rs = np.random.RandomState(23)
    checked = 0
    for it in range(60):
        t, cap = random_table(rs)
        world, dp = [(2, 1), (4, 1), (4, 2), (8, 2)][it % 4]
        sp = world // dp
        gbs = dp * int(rs.randint(1, 3))
        try:
            o = oplan.plan_step(t, cap, gbs, dp, sp, world, 1, "lpt")
        except ValueError:
            continue
        thr = int(rs.randint(0, cap + 1))
        c = ocph.place(o, t, gbs, dp, sp, cap, thr)
        me = int(rs.randint(0, world))
        d = cp_device_plan(t, cap, gbs, dp, sp, world, me, "lpt", thr)
        assert_cp_equal(d, c, t, me)
        g = int(rs.choice([x for x in (1, 2, 4) if world % x == 0]))
        eta = int(rs.randint(0, cap + 1))
        lay = olssp.layout(c, t["lens"], world, eta, g)
        d = cp_device_plan(t, cap, gbs, dp, sp, world, me, "lpt", thr, g, eta)
        assert_lssp_equal(d, c, lay, t, me)
        checked += 1
    assert checked > 25


@pytest.mark.parametrize("reshard", ["ulysses", "cp_hybrid"])
def test_text_segments_match_oracle(cuda_device, reshard):
    from oracle import cphybrid as ocph
    n = 0
    for name, st, t, _ in golden_steps():
        for world, dp in ((1, 1), (2, 2), (4, 2), (4, 1)):
            sp = world // dp
            gbs = st["gbs"] * dp // st["dp"] if st["gbs"] % st["dp"] == 0 else st["gbs"]
            try:
                o = oplan.plan_step(t, configs.CAPACITY, gbs, dp, sp, world, 1, "lpt")
            except ValueError:
                continue
            if reshard == "cp_hybrid":
                o = ocph.place(o, t, gbs, dp, sp, configs.CAPACITY)
            table = to_table(t)
            for me in range(world):
                cfg = planner.make_cfg(table, configs.CAPACITY, gbs, dp, sp, world, 1, "lpt",
                                       False, me, reshard=reshard, text_embed=True)
                plan = planner.plan_step(planner.DeviceTable(table, "cuda"), cfg)
                plan.check(table)
                d = plan.host()
                toff = odp.text_offsets(t)
                text = toff >= 0
                assert np.array_equal(d["text_off"][text], toff[text])
                assert np.array_equal(d["tseg"], odp.text_by_rank(o, t, me))
                assert np.array_equal(d["rseg"], odp.pieces_by_rank(o, me))
                n += 1
    assert n > 20


def test_plan_at_the_sample_limit(cuda_device):
    """4096 samples (the device planner's limit) plan bit-exactly; 4097 is refused
    with a ValueError before any launch."""
    rs = np.random.RandomState(8)
    n = 4096
    lens = rs.randint(1, 600, size=n)
    t = dict(lens=lens, mods=rs.randint(0, 4, size=n), ids=rs.permutation(n),
             carry_seq=np.zeros(0, np.int64), n_carry_seqs=0,
             chunk_off=[0, 1500, 3000, n])
    o = oplan.plan_step(t, 16384, 8, 8, 1, 8, 1, "lpt")
    for me in (0, 7):
        d = device_plan(t, 16384, 8, 8, 1, 8, me, "lpt")
        assert_plan_equal(d, o, t, me)
    t2 = dict(t, lens=np.append(lens, 5), mods=np.append(t["mods"], 1),
              ids=np.append(t["ids"], n), chunk_off=[0, 1500, 3000, n + 1])
    with pytest.raises(ValueError, match="4096"):
        device_plan(t2, 16384, 8, 8, 1, 8, 0, "lpt")


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_assemble_table_matches_oracle(cuda_device, world):
    """mux_assemble_table (csrc/meta.cu) on the records of every rank's share
    rebuilds the centralized step table bit for bit; its device plan equals
    the oracle's (the decentralized metadata all-gather)."""
    import torch
    cap, capc = 2048, 64
    n = 0
    for name, st, t, _ in golden_steps():
        if st["step"] > 1:
            continue
        table = to_table(t)
        recs = np.stack([table.shard(r, world).record(cap, capc) for r in range(world)])
        want = oplan.assemble_records(list(recs), cap, capc)
        blob = torch.full((table.blob().size + 4,), -7, dtype=torch.int64, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        dev = torch.from_numpy(recs.reshape(-1)).cuda()
        _lib_ = planner._lib
        _lib_.check(_lib_.lib().mux_assemble_table(dev.data_ptr(), world, cap, capc,
                                                   blob.data_ptr(), blob.numel(),
                                                   err.data_ptr(),
                                                   torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert int(err.item()) == 0
        assert np.array_equal(blob.cpu().numpy()[:table.blob().size], table.blob())
        for k in ("lens", "ids", "carry_seq"):
            assert np.array_equal(want[k], np.asarray(t[k]))
        n += 1
    assert n >= 4
    # world 1 through gather_table (no process group): the plan of the gathered table
    for name, st, t, _ in golden_steps():
        if st["world"] == 1 and st["step"] == 0:
            dt = planner.gather_table(to_table(t), "cuda")
            cfg = planner.make_cfg(dt.table, configs.CAPACITY, st["gbs"], 1, 1, 1)
            plan = planner.plan_step(dt, cfg)
            plan.check(dt.table)
            assert_plan_equal(plan.host(), oracle_plan(t, st), t, 0)


@pytest.mark.parametrize("rg,sp_enc", [(4, 2), (4, 4), (2, 2), (8, 4)])
def test_lssp_inside_reorder_groups_matches_oracle(cuda_device, rg, sp_enc):
    """LSSP groups nested in reorder groups (the planner requires rg % sp_enc == 0):
    every rank's LSSP layout and segment tables bit-exact against the oracle."""
    from oracle import lssp as olssp
    n = 0
    for name, st, t, _ in golden_steps():
        world, dp = st["world"], st["dp"]
        if world < rg or world % rg:
            continue
        o = oplan.plan_step(t, configs.CAPACITY, st["gbs"], dp, world // dp, world, 1,
                            "lpt_local", reorder_group=rg)
        lay = olssp.layout(o, t["lens"], world, 2048, sp_enc)
        for me in range(world):
            d = lssp_device_plan(t, configs.CAPACITY, st["gbs"], dp, world // dp, world, me,
                                 "lpt_local", sp_enc, 2048, reorder_group=rg)
            assert_lssp_equal(d, o, lay, t, me)
            n += 1
    assert n >= 4


def test_cp_hybrid_with_reorder_groups_and_flops_costs(cuda_device):
    """CpHybrid LLM placement on top of an encoder plan balanced inside reorder
    groups of 2 with the flops cost: every rank bit-exact against the oracle."""
    from oracle import cphybrid as ocph
    n = 0
    for name, st, t, _ in golden_steps():
        for world, dp in ((4, 1), (4, 2), (8, 2)):
            sp = world // dp
            gbs = st["gbs"] * dp // st["dp"] if st["gbs"] % st["dp"] == 0 else st["gbs"]
            try:
                o = oplan.plan_step(t, configs.CAPACITY, gbs, dp, sp, world, 1, "lpt_local",
                                    reorder_group=2, cost=FLOPS)
            except ValueError:
                continue
            c = ocph.place(o, t, gbs, dp, sp, configs.CAPACITY, 0)
            for me in range(world):
                d = cp_device_plan(t, configs.CAPACITY, gbs, dp, sp, world, me, "lpt_local", 0,
                                   reorder_group=2, cost=FLOPS)
                assert_cp_equal(d, c, t, me)
                n += 1
    assert n > 8
