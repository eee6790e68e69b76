"""CPU oracle for the encoder<->LLM data path — TEST INFRASTRUCTURE ONLY.

Nothing in `paper_2605_08962_b200` imports this package.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
leg may import it, and there only as the checker or the timed CPU baseline,
never as the thing measured or shipped.

Parity anchors:
* `workload.py` here restates the reference generator and packer
  (/root/reference/pkg/src/muxsim/workload.py) and is pinned against golden
  vectors produced by the reference itself (tests/golden/make_golden.py).
* `planner.py` restates SPEC-only operations (kk_partition, grouped_reorder,
  restore_order, plan_reshard) and is pinned by the SPEC's known-answer tests
  (SPEC.md:85-96, :396-398, :405-407, :468-469).  The data-plane layout
  (loader arena order, encoder order, LLM positions) has no reference code:
  for those parts parity is "unpinned" by the reference and defined here.
* `dataplane.py` is the fake-world (all ranks in one process) data movement.
"""
