"""B200-native label-partitioned DC-CGAN training step (arXiv 2102.10485).

Native library: paper_2102_10485_b200/_lib/libpartgan_b200.so (sm_100a
kernels + C++ host), bound here through ctypes.  See DESIGN.md.
"""
from . import _native
from .archs import CONFIGS, Arch, algorithmic_flops_per_image, baseline_arch
from .trainer import (AdamConfig, GroupSpec, LabelGroup, StepReport, cosine_label, derive_seed, estimate_priors,
                      make_group, partition_by_label, shard_begin)

__all__ = [
    "_native", "CONFIGS", "Arch", "algorithmic_flops_per_image", "baseline_arch", "AdamConfig", "GroupSpec",
    "LabelGroup", "StepReport", "cosine_label", "derive_seed", "estimate_priors", "make_group", "partition_by_label",
    "shard_begin",
]
