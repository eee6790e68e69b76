"""Shared test helpers: golden fixtures -> step tables, oracle plans."""

from __future__ import annotations

import json
import os

import numpy as np

from oracle import planner as oplan
from oracle import workload as owork
from paper_2605_08962_b200 import configs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MOD = {"text": 0, "image": 1, "video": 2, "audio": 3}


def golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def golden_steps():
    """Yield (config, step record, table dict, modality map) for every golden step."""
    G = golden("configs.json")
    for name, rec in G.items():
        if not isinstance(rec, dict) or rec["toy"]:
            continue
        seen = {}
        for st in rec["steps"]:
            for s in st["drawn"]:
                seen[s[0]] = s[1]
            carry = [[tuple(x) for x in q] for q in st["carry_in"]]
            # chunk sizes: regenerate with the oracle (pinned to the same golden)
            cfg = configs.CONFIGS[name]
            descs = owork.descs_from_config(configs.DATASETS, cfg["datasets"])
            _, _, drawn, chunks = owork.generate(descs, cfg["phases"], cfg["interp"] == "linear",
                                                 st["step"], cfg["seed"], st["gbs"], st["dp"], 1,
                                                 configs.CAPACITY, carry or None)
            table = oplan.step_table(carry, drawn, chunks, seen)
            yield name, st, table, seen


def oracle_plan(table, st, method="lpt", pooled=False):
    world, dp = st["world"], st["dp"]
    return oplan.plan_step(table, configs.CAPACITY, st["gbs"], dp, world // dp, world, 1,
                           method, pooled)


def random_table(rs, S=None, n_chunks=None, cap=None, n_carry_seqs=None):
    """A random step table with carry sequences and several chunks."""
    cap = cap or int(rs.choice([64, 256, 1024]))
    ncs = int(rs.randint(0, 4)) if n_carry_seqs is None else n_carry_seqs
    lens, mods, ids, cseq = [], [], [], []
    nid = 0
    for q in range(ncs):
        fill = 0
        for _ in range(int(rs.randint(1, 5))):
            L = int(rs.randint(0, max(cap // 3, 2)))
            if fill + L > cap:
                break
            fill += L
            lens.append(L); mods.append(int(rs.randint(0, 4))); ids.append(nid); cseq.append(q)
            nid += 1
        if not cseq or cseq[-1] != q:   # every carry sequence has >= 1 span
            lens.append(1); mods.append(1); ids.append(nid); cseq.append(q); nid += 1
    off = [len(lens)]
    for _ in range(n_chunks if n_chunks is not None else int(rs.randint(1, 4))):
        n = int(rs.randint(1, S or 80))
        for _ in range(n):
            lens.append(int(rs.randint(0 if rs.rand() < 0.1 else 1, cap + 1)))
            mods.append(int(rs.randint(0, 4)))
            ids.append(nid if rs.rand() > 0.1 else int(rs.randint(0, nid + 1)))
            nid += 1
        off.append(len(lens))
    return dict(lens=np.array(lens, np.int64), mods=np.array(mods, np.int64),
                ids=np.array(ids, np.int64), carry_seq=np.array(cseq, np.int64),
                n_carry_seqs=ncs, chunk_off=off), cap
