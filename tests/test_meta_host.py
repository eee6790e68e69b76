"""Decentralized metadata records on the host (no GPU): every rank's share of a
step (StepTable.shard) packed into a record (StepTable.record) and assembled in
rank order (oracle.planner.assemble_records) is the centralized step table again,
for random tables with carried sequences and chunks, world sizes 1..8 — including
more ranks than chunks or carried sequences (empty shares) — and the plan of the
assembled table equals the centralized plan."""

import numpy as np
import pytest

from oracle import planner as oplan
from tests.helpers import random_table
from tests.test_gpu_planner import to_table


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_shards_reassemble_to_the_table(world):
    rs = np.random.RandomState(100 + world)
    for _ in range(25):
        t, cap = random_table(rs, S=40, n_chunks=int(rs.randint(1, 4)))
        table = to_table(t)
        recs = [table.shard(r, world).record(256, 16) for r in range(world)]
        got = oplan.assemble_records(recs, 256, 16)
        for k in ("lens", "mods", "ids", "carry_seq"):
            assert np.array_equal(got[k], np.asarray(t[k])), k
        assert list(got["chunk_off"]) == list(t["chunk_off"])
        assert got["n_carry_seqs"] == t["n_carry_seqs"]
        shard_rows = sum(table.shard(r, world).S for r in range(world))
        assert shard_rows == table.S  # a partition of the step's rows


def test_record_capacity_is_checked():
    rs = np.random.RandomState(3)
    t, _ = random_table(rs, S=60, n_chunks=3)
    table = to_table(t)
    with pytest.raises(ValueError, match="exceeds the record capacity"):
        table.record(4, 16)
