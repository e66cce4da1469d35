"""The reference driver's JSON run configuration (include/partgan/run.hpp:35-58,
src/run.cpp:71-141 validate / config_from_json) for the device path: the same
key set, unknown keys rejected with the reference's message ("unknown config
key '<prefix><key>'"), the same validation rules and messages.  Deliberate
narrowing to what the B200 path trains:
  - mode: "distributed-cgan" only (the paper's label-partitioned method);
  - arch: "auto" | "c1" | "c2" | "c3" | "c4" (the BASELINE.json architectures;
    "auto" picks from the synthetic image size);
  - dataset: kind "synthetic" with synthetic.kind "cosine-field" (the BASELINE
    synthetic data; no IDX / CIFAR files exist in this environment).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field, asdict


class ConfigError(RuntimeError):
    """run.hpp:16 ConfigError (the CLI maps it to exit code 2)."""


TOP_KEYS = ("dataset", "mode", "d_z", "epochs", "batch_size", "lr", "beta1", "beta2", "adam_eps", "bn_eps",
            "bn_momentum", "clamp", "init_std", "seed", "workers", "arch", "hidden", "sigmoid_output", "out_dir")
DATASET_KEYS = ("kind", "images", "labels", "pad_to_32", "paths", "synthetic")
SYNTHETIC_KEYS = ("kind", "k", "per_class_n", "seed", "means", "stddev", "image_size")
ARCH_BY_SIZE = {28: "c1", 32: "c2", 64: "c4"}


@dataclass
class SyntheticSpec:
    kind: str = "cosine-field"
    k: int = 10
    per_class_n: int = 256
    seed: int = 2024
    stddev: float = 0.1
    image_size: int = 28


@dataclass
class DatasetConfig:
    kind: str = "synthetic"
    synthetic: SyntheticSpec = field(default_factory=SyntheticSpec)


@dataclass
class RunConfig:
    dataset: DatasetConfig = field(default_factory=DatasetConfig)
    mode: str = "distributed-cgan"
    d_z: int = 100
    epochs: int = 50
    batch_size: int = 64
    lr: float = 2e-4
    beta1: float = 0.5
    beta2: float = 0.999
    adam_eps: float = 1e-8
    bn_eps: float = 1e-5
    bn_momentum: float = 0.1
    clamp: float = 1e-7
    init_std: float = 0.02
    seed: int = 1234
    workers: int = 0
    arch: str = "auto"
    hidden: int = 128
    sigmoid_output: bool = True
    out_dir: str = "run-out"

    def validate(self) -> None:
        """run.cpp:71-90, with the device path's arch / mode / dataset sets."""
        if self.d_z < 1:
            raise ConfigError("d_z must be >= 1")
        if self.epochs < 1:
            raise ConfigError("epochs must be >= 1")
        if self.batch_size < 1:
            raise ConfigError("batch_size must be >= 1")
        if self.lr < 0:
            raise ConfigError("lr must be >= 0")
        if not (0 <= self.beta1 < 1) or not (0 <= self.beta2 < 1):
            raise ConfigError("betas must lie in [0, 1)")
        if not self.adam_eps > 0:
            raise ConfigError("adam_eps must be > 0")
        if not self.bn_eps > 0:
            raise ConfigError("bn_eps must be > 0")
        if not 0 <= self.bn_momentum <= 1:
            raise ConfigError("bn_momentum must lie in [0, 1]")
        if not 0 < self.clamp < 0.5:
            raise ConfigError("clamp must lie in (0, 0.5)")
        if not self.init_std > 0:
            raise ConfigError("init_std must be > 0")
        if self.workers < 0:
            raise ConfigError("workers must be >= 0")
        if self.hidden < 1:
            raise ConfigError("hidden must be >= 1")
        if self.arch not in ("auto", "c1", "c2", "c3", "c4"):
            raise ConfigError(f"unknown arch '{self.arch}' (expected auto | c1 | c2 | c3 | c4)")
        if not self.out_dir:
            raise ConfigError("out_dir must be non-empty")
        if self.dataset.kind != "synthetic":
            raise ConfigError(f"unknown dataset kind '{self.dataset.kind}'" if self.dataset.kind not in ("idx", "cifar")
                              else f"dataset kind '{self.dataset.kind}' needs files that do not exist here")
        if self.mode != "distributed-cgan":
            raise ConfigError(f"unknown mode '{self.mode}' (the B200 path trains distributed-cgan)")
        if self.dataset.synthetic.kind != "cosine-field":
            raise ConfigError(f"unknown synthetic kind '{self.dataset.synthetic.kind}'")
        if self.arch == "auto" and self.dataset.synthetic.image_size not in ARCH_BY_SIZE:
            raise ConfigError(f"no architecture for image_size {self.dataset.synthetic.image_size} (28, 32 or 64)")

    def resolved_arch(self) -> int:
        a = self.arch if self.arch != "auto" else ARCH_BY_SIZE[self.dataset.synthetic.image_size]
        return int(a[1:])


def _check_keys(d: dict, prefix: str, allowed) -> None:
    for k in d:
        if k not in allowed:
            raise ConfigError(f"unknown config key '{prefix}{k}'")


def config_from_json(j: dict) -> RunConfig:
    """run.cpp:92-141: unknown keys rejected at every level."""
    if not isinstance(j, dict):
        raise ConfigError("config must be a JSON object")
    _check_keys(j, "", TOP_KEYS)
    cfg = RunConfig()
    for k in TOP_KEYS:
        if k in j and k != "dataset":
            want = type(getattr(cfg, k))
            v = j[k]
            if want is float and isinstance(v, int):
                v = float(v)
            if not isinstance(v, want) or (want is int and isinstance(v, bool)):
                raise ConfigError(f"config key '{k}' must be {want.__name__}")
            setattr(cfg, k, v)
    cfg.mode = cfg.mode.replace("_", "-")
    if "dataset" in j:
        d = j["dataset"]
        _check_keys(d, "dataset.", DATASET_KEYS)
        if "kind" in d:
            cfg.dataset.kind = d["kind"]
        if "synthetic" in d:
            s = d["synthetic"]
            _check_keys(s, "dataset.synthetic.", SYNTHETIC_KEYS)
            for k in ("kind", "k", "per_class_n", "seed", "stddev", "image_size"):
                if k in s:
                    setattr(cfg.dataset.synthetic, k, s[k])
            if "means" in s:
                raise ConfigError("dataset.synthetic.means applies to the blob kinds, not cosine-field")
    cfg.validate()
    return cfg


def load_config_file(path: str) -> RunConfig:
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise ConfigError(f"cannot read config file {path}: {e}") from None
    except json.JSONDecodeError as e:
        raise ConfigError(f"{path}: invalid JSON: {e}") from None
    return config_from_json(j)


def config_to_json(cfg: RunConfig) -> dict:
    return asdict(cfg)
