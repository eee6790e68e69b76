"""Host-side logic of the product package (no GPU): generator, batching, costs, C ABI load."""

import json
import os
import re

import numpy as np
import pytest

from paper_2605_08962_b200 import _lib, configs, workload as W
from tests.helpers import golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sample_step_matches_reference_golden():
    G = golden("configs.json")
    reg, sched = configs.build(W, "cfg1")
    chunk = W.sample_step(reg, sched, 0, 64, 1234)
    assert [[s.id, s.modality.value, s.dataset, s.length] for s in chunk] == G["cfg1"]["samples"]
    for name in ("cfg2", "cfg4", "cfg5"):
        reg, sched = configs.build(W, name)
        st = G[name]["steps"][0]
        cfg = configs.CONFIGS[name]
        # first drawn chunk of step 0 (size from generate_batch's draw rule)
        mean = np.mean([reg.get(n).mean_len for n, r in sched.recipe_at(0).entries if r > 0])
        n = max(int((st["gbs"] + 1) * configs.CAPACITY / mean) + 1, 16)
        chunk = W.sample_step(reg, sched, 0, n, cfg["seed"], 0)
        assert [[s.id, s.modality.value, s.dataset, s.length] for s in chunk] == st["drawn"][:n]


def test_recipe_at_matches_reference_golden():
    M = golden("misc.json")
    sched = W.PhaseSchedule(((0, W.MixtureRecipe.of(image=0.5, text=0.5)),
                             (1000, W.MixtureRecipe.of(image=0.13, audio=0.74, text=0.13))),
                            W.Interpolation.LINEAR)
    for step, entries in M["recipes"].items():
        assert [list(e) for e in sched.recipe_at(int(step)).entries] == entries


def test_build_global_batch_matches_reference_golden():
    M = golden("misc.json")
    for rec in M["build_global_batch"]:
        seqs = [W.PackedSequence(16, [(i, i + 1)]) for i in range(rec["n"])]
        res = rec["result"]
        try:
            b, rest = W.build_global_batch(seqs, 0, rec["gbs"], rec["dp"], rec["mbs"])
        except W.ConfigError as e:
            assert res["error"] == "ConfigError" and str(e) == res["message"]
            continue
        except ValueError as e:
            assert res["error"] == "ValueError" and str(e) == res["message"]
            continue
        assert len(b.sequences) == res["batch"] and len(rest) == res["carry"]
        assert b.microbatches_per_replica == res["mbs_per_replica"]
        got = [[[sp[0] for q in b.replica_microbatch(r, m) for sp in q.spans]
                for m in range(b.microbatches_per_replica)] for r in range(rec["dp"])]
        assert got == res["replica_mb"]


def test_config_errors_match_reference():
    with pytest.raises(W.ConfigError):
        W.DatasetDescriptor("x", W.Modality.TEXT, 0.0, 10)
    with pytest.raises(W.ConfigError):
        W.MixtureRecipe.of(a=0.5)
    with pytest.raises(W.ConfigError):
        W.PhaseSchedule(((1, W.MixtureRecipe.of(a=1.0)),))
    reg = W.DatasetRegistry([W.DatasetDescriptor("a", W.Modality.TEXT, 10.0, 100)])
    sched = W.PhaseSchedule(((0, W.MixtureRecipe.of(b=1.0)),))
    with pytest.raises(W.ConfigError):
        W.sample_step(reg, sched, 0, 4, 0)
    with pytest.raises(ValueError):
        W.sample_step(reg, W.PhaseSchedule(((0, W.MixtureRecipe.of(a=1.0)),)), -1, 4, 0)


def test_export_batch_schema(tmp_path):
    b = W.GlobalBatch(3, [W.PackedSequence(16, [(1, 5), (2, 4)])], 1, 1)
    samples = {1: W.Sample(1, W.Modality.IMAGE, "x", 5)}
    W.export_batch(b, samples, tmp_path / "b.jsonl")
    rec = json.loads((tmp_path / "b.jsonl").read_text())
    assert rec == {"capacity": 16, "fill": 9, "schema_version": 1, "sequence": 0, "step": 3,
                   "spans": [{"modality": "image", "sample": 1, "tokens": 5},
                             {"modality": None, "sample": 2, "tokens": 4}]}


def test_export_batch_matches_reference_bytes(tmp_path):
    """export_batch JSONL byte-identical to the reference's (tests/golden/export.json,
    written by the reference's own export_batch on two chained cfg5 steps)."""
    from tests.helpers import golden
    for rec in golden("export.json")["batches"]:
        seqs = [W.PackedSequence(rec["capacity"], [tuple(sp) for sp in q]) for q in rec["seqs"]]
        b = W.GlobalBatch(rec["step"], seqs, rec["dp"], rec["mbs"])
        samples = {i: W.Sample(i, W.Modality(m), d, L) for i, m, d, L in rec["samples"]}
        out = tmp_path / f"b{rec['step']}.jsonl"
        W.export_batch(b, samples, out)
        assert out.read_text() == rec["jsonl"]


def test_capi_exports_every_declared_symbol():
    from paper_2605_08962_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "mux_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|void|const char\*|size_t)\s+(mux_\w+)\(", hdr, re.M))
    assert declared, "no declarations parsed"
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_lib.EXPORTS)
    assert L.mux_version() == 3


def test_plan_layout_on_cpu():
    from paper_2605_08962_b200 import planner
    t = planner.StepTable(np.array([5, 3], np.int32), np.array([1, 0], np.int32),
                          np.array([1, 2], np.int64), np.zeros(0, np.int32), 0,
                          np.array([0, 2], np.int32))
    cfg = planner.make_cfg(t, 16, gbs=1)
    L = planner.layout_of(cfg)
    assert L.total > 0 and L.total % 256 == 0
    cfg.S = 100000
    with pytest.raises(ValueError):
        planner.layout_of(cfg)


def test_ctypes_struct_mirrors_match_the_library():
    """The ctypes mirrors of mux_plan_cfg / mux_plan_layout / mux_proj_group have
    the C sizes (no GPU needed: mux_abi_sizes is host code)."""
    import ctypes as C
    out = (C.c_int64 * 3)()
    _lib.lib().mux_abi_sizes(out)
    assert list(out) == [C.sizeof(_lib.PlanCfg), C.sizeof(_lib.PlanLayout),
                         C.sizeof(_lib.ProjGroup)]


def test_header_is_plain_c99(tmp_path):
    """include/mux_b200.h is a C ABI: it compiles as strict C99 (no C++ or CUDA types)
    and a C program linking libmuxb200.so sees the same struct sizes as ctypes."""
    import ctypes as C
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    src = tmp_path / "t.c"
    src.write_text(
        '#include <stdio.h>\n#include "mux_b200.h"\n'
        "int main(void) { printf(\"%zu %zu %zu\\n\", sizeof(mux_plan_cfg),"
        " sizeof(mux_plan_layout), sizeof(mux_proj_group)); return mux_version() > 0 ? 0 : 1; }\n")
    exe = tmp_path / "t"
    libdir = os.path.join(ROOT, "paper_2605_08962_b200")
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror",
                        "-I", os.path.join(ROOT, "include"), str(src), "-L", libdir,
                        "-lmuxb200", "-Wl,-rpath," + libdir, "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert [int(x) for x in out.stdout.split()] == [
        C.sizeof(_lib.PlanCfg), C.sizeof(_lib.PlanLayout), C.sizeof(_lib.ProjGroup)]


def test_integration_stub_mirrors_the_abi():
    """The ctypes stub printed in INTEGRATION.md §2 (what the reference package
    would add) mirrors mux_plan_cfg / mux_plan_layout of this build."""
    import ctypes as C
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = next(b.split("```", 1)[0] for b in text.split("```python")[1:] if "class PlanCfg" in b)
    body = code[code.index("class PlanCfg"):code.index("def hybrid_pack")]
    ns = {"ctypes": C}
    exec(body, ns)
    out = (C.c_int64 * 3)()
    _lib.lib().mux_abi_sizes(out)
    assert C.sizeof(ns["PlanCfg"]) == out[0]
    assert C.sizeof(ns["PlanLayout"]) == out[1]
