"""Cost formulas on the data path (reference: pkg/src/muxsim/costs.py).

Only the parts the hot path uses: the per-sample encoder cost that can weight
the rebalance (flops_forward, costs.py:108-124), and the collective byte
accounting (volume_factor / comm_time, costs.py:84-105), kept as the modeled
comparator for the measured NVLink exchange.  The memory/offload model
(costs.py:131-189) is out of scope.

Plus the algorithmic byte/FLOP counts of the B200 kernels,
used by bench.py for the roofline.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

COLLECTIVES = ("all_gather", "all_to_all", "all_reduce", "reduce_scatter", "broadcast", "p2p")


class ModelKind(str, Enum):
    ENCODER = "encoder"
    LLM = "llm"


@dataclass(frozen=True)
class ModelSpec:
    name: str
    kind: ModelKind
    params: float
    layers: int
    hidden: int
    heads: int
    modality: str = ""
    tokens_per_patch: int = 588
    flops_multiplier: float = 1.0

    def __post_init__(self):
        if self.params <= 0:
            raise ValueError(f"model {self.name}: params must be positive")
        if self.layers < 1:
            raise ValueError(f"model {self.name}: layers must be >= 1")
        if self.hidden % max(self.heads, 1) != 0:
            raise ValueError(f"model {self.name}: heads must divide hidden")


@dataclass(frozen=True)
class LinkParams:
    latency_s: float
    bytes_per_s: float

    def __post_init__(self):
        if self.latency_s <= 0 or self.bytes_per_s <= 0:
            raise ValueError("link latency and bandwidth must be positive")


@dataclass(frozen=True)
class CommModel:
    intra: LinkParams = LinkParams(5e-6, 200e9)
    inter: LinkParams = LinkParams(10e-6, 50e9)
    primitive_overhead_s: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.intra.bytes_per_s < self.inter.bytes_per_s:
            raise ValueError("intra-node links must not be slower than inter-node links")
        bad = [p for p in self.primitive_overhead_s if p not in COLLECTIVES]
        if bad:
            raise ValueError(f"unknown collective primitive {bad[0]!r}")


def volume_factor(primitive: str, group_size: int) -> float:
    """Per-rank wire bytes / payload: 1 for p2p, (g-1)/g for collectives."""
    if primitive not in COLLECTIVES:
        raise ValueError(f"unknown collective primitive {primitive!r}")
    if primitive == "p2p":
        return 1.0
    g = max(group_size, 1)
    return 0.0 if g == 1 else (g - 1) / g


def comm_time(model: CommModel, primitive: str, nbytes: int, group_size: int,
              intra_node: bool) -> float:
    """Alpha-beta seconds for one collective of `nbytes` per rank."""
    if nbytes < 0:
        raise ValueError("nbytes must be nonnegative")
    if group_size < 1:
        raise ValueError("group must be nonempty")
    link = model.intra if intra_node else model.inter
    return (link.latency_s + model.primitive_overhead_s.get(primitive, 0.0)
            + nbytes * volume_factor(primitive, group_size) / link.bytes_per_s)


def flops_forward(spec: ModelSpec, tokens: int, seq_len: int) -> float:
    """2*params*tokens + 2*layers*hidden*tokens*seq_len, times the multiplier."""
    if tokens < 0:
        raise ValueError("tokens must be nonnegative")
    if seq_len < 1:
        raise ValueError("seq_len must be >= 1")
    if tokens == 0:
        return 0.0
    dense = 2.0 * spec.params * tokens
    attention = 2.0 * spec.layers * spec.hidden * tokens * seq_len
    return (dense + attention) * spec.flops_multiplier


def encoder_cost_params(spec: ModelSpec) -> tuple[float, float]:
    """(lin, quad) of the device planner's flops cost model (mux_plan_cfg
    cost_model = MUX_COST_FLOPS): lin L + quad L^2 == flops_forward(spec, L, L)
    bit for bit (an encoder's seq_len is the sample length, costs.py:112-114),
    which needs integer-valued params/layers/hidden and multiplier 1 so that
    every cost and load sum stays an exact fp64 integer on every rank."""
    if spec.flops_multiplier != 1.0 or float(spec.params) != int(spec.params):
        raise ValueError("the device cost model needs integer params and flops_multiplier 1")
    return 2.0 * spec.params, 2.0 * spec.layers * spec.hidden


def flops_backward(spec: ModelSpec, tokens: int, seq_len: int) -> float:
    return 2.0 * flops_forward(spec, tokens, seq_len)


# --------------------------------------------------------------------------
# algorithmic traffic of the B200 kernels
# --------------------------------------------------------------------------

def pack_bytes(rows: int, d_in: int) -> int:
    """Pack/dispatch: read + write of every loader row (2 B per bf16)."""
    return 2 * rows * d_in * 2


def scatter_bytes(rows: int, d_row: int) -> int:
    """Return/scatter with rows already LLM-wide: read + write."""
    return 2 * rows * d_row * 2


def projector_flops(rows: int, d_enc: int, d_llm: int) -> int:
    return 2 * rows * d_enc * d_llm


def projector_bytes(rows: int, d_enc: int, d_llm: int) -> int:
    """Read X, write Y, read W once."""
    return rows * d_enc * 2 + rows * d_llm * 2 + d_enc * d_llm * 2
