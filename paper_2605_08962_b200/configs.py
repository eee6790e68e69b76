"""Workload configurations for the encoder<->LLM data path.

Plain data only, so that the same table can build objects from this package,
from the CPU oracle, or (in this container only) from the reference's own
``muxsim.workload`` module when golden vectors are regenerated.

Dataset means come from the paper; capacity 16384
from SPEC.md:57.  Widths: 588 = 3*14*14 pixels per visual token
(pkg/src/muxsim/costs.py:42); audio 512, video-as-patch-rows and d_enc/d_llm
are the builder's choices recorded in SURVEY.md §8.1-9.
"""

from __future__ import annotations

CAPACITY = 16384

# name -> (modality value, mean_len, max_len)
DATASETS = {
    "openimages": ("image", 3800.0, CAPACITY),
    "refcocog": ("image", 1400.0, CAPACITY),
    "video": ("video", 4096.0, CAPACITY),
    "librispeech": ("audio", 340.0, CAPACITY),
    "text": ("text", 1000.0, CAPACITY),
    "bytedlong": ("text", 6000.0, CAPACITY),
}

# Modality codes used on the device (same order as workload.Modality).
MOD_CODE = {"text": 0, "image": 1, "video": 2, "audio": 3}
# Encoder group per modality: image/video share the ViT, audio has its own.
GROUP_OF_MOD = {0: -1, 1: 0, 2: 0, 3: 1}
N_GROUPS = 2

# Per-encoder-group widths (bf16 elements per token row).
D_IN = (588, 512)      # vision patch row, audio mel-stack row
D_ENC = (1280, 1280)   # ViT-600M-shaped / audio encoder hidden
D_LLM = 4096           # 7B-shaped LLM hidden

# Encoder shapes per group for the optional flops-weighted rebalance
# (costs.flops_forward, pkg/src/muxsim/costs.py:108-124): (params, layers,
# hidden).  ViT-600M-shaped: 32 layers x 1280 hidden (12 h^2 per layer); the
# audio encoder is given the same shape (builder's choice).
ENCODER_SHAPES = ((32 * 12 * 1280 * 1280, 32, 1280), (32 * 12 * 1280 * 1280, 32, 1280))

_CFG5_PHASES = (
    {"openimages": 0.13, "video": 0.0, "librispeech": 0.74, "text": 0.13},
    {"openimages": 0.55, "video": 0.10, "librispeech": 0.0, "text": 0.35},
    {"openimages": 0.40, "video": 0.30, "librispeech": 0.10, "text": 0.20},
)


def _cycling(phases, n_steps=100):
    return tuple((s, phases[s % len(phases)]) for s in range(n_steps))


# Each config: datasets, phase table [(start_step, {dataset: ratio})],
# interpolation, seed, gbs-per-replica, llm sp, projector, carryover chaining.
CONFIGS = {
    # configs[0]: CPU toy; one sample_step(n=64) packed whole.
    "cfg1": dict(datasets=("openimages", "text"),
                 phases=((0, {"openimages": 0.5, "text": 0.5}),),
                 interp="step", seed=1234, toy_n=64, gbs_per_replica=None,
                 sp=1, projector=False, carry=False),
    # configs[1]: ViT-600M -> 7B, 64K-token image-text batch, projector fused.
    "cfg2": dict(datasets=("openimages", "text"),
                 phases=((0, {"openimages": 0.5, "text": 0.5}),),
                 interp="step", seed=1234, gbs_per_replica=4,
                 sp=1, projector=True, carry=True),
    # configs[2]: image + video with 2.71x intra-image skew at 2/4/8 GPUs.
    "cfg3": dict(datasets=("openimages", "refcocog", "video", "text"),
                 phases=((0, {"openimages": 0.3, "refcocog": 0.2,
                              "video": 0.3, "text": 0.2}),),
                 interp="step", seed=2605, gbs_per_replica=2,
                 sp=1, projector=False, carry=True),
    # configs[3]: audio + long text (17.6x disparity), LLM dp=2 x Ulysses sp=4.
    "cfg4": dict(datasets=("librispeech", "bytedlong"),
                 phases=((0, {"librispeech": 0.7, "bytedlong": 0.3}),),
                 interp="step", seed=2605, gbs_per_replica=8,
                 sp=4, projector=False, carry=True),
    # north_star target-1: mixed image/video/audio/text, projector off, 1 GPU.
    "target1": dict(datasets=("openimages", "video", "librispeech", "text"),
                    phases=((0, _CFG5_PHASES[2]),),
                    interp="step", seed=2605, gbs_per_replica=4,
                    sp=1, projector=False, carry=True),
    # configs[4]: phase changes every step, 16 x 16384 tokens at 8 GPUs.
    "cfg5": dict(datasets=("openimages", "video", "librispeech", "text"),
                 phases=_cycling(_CFG5_PHASES),
                 interp="step", seed=2605, gbs_per_replica=2,
                 sp=1, projector=False, carry=True),
}


def build(mod, name):
    """Build (registry, schedule) for config `name` from a workload-like module.

    `mod` must expose DatasetDescriptor, Modality, DatasetRegistry,
    MixtureRecipe, PhaseSchedule and Interpolation with the reference's
    signatures (pkg/src/muxsim/workload.py:37-206).
    """
    cfg = CONFIGS[name]
    descs = []
    for ds in cfg["datasets"]:
        modality, mean, max_len = DATASETS[ds]
        descs.append(mod.DatasetDescriptor(ds, mod.Modality(modality), mean, max_len))
    reg = mod.DatasetRegistry(descs)
    phases = tuple((s, mod.MixtureRecipe.of(**r)) for s, r in cfg["phases"])
    sched = mod.PhaseSchedule(phases, mod.Interpolation(cfg["interp"]))
    return reg, sched
