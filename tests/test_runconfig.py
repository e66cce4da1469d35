"""The reference JSON RunConfig (run.hpp:35-58, run.cpp:71-141) on the device
CLI: unknown keys rejected at every level with the reference's message, the
reference's validation messages, ConfigError -> exit code 2, and
estimate_priors (partition.cpp:58-74).  CPU only (no training)."""
import json
import subprocess
import sys

import numpy as np
import pytest

from paper_2102_10485_b200 import estimate_priors
from paper_2102_10485_b200.runconfig import ConfigError, config_from_json


def test_unknown_keys_rejected_at_every_level():
    with pytest.raises(ConfigError, match="unknown config key 'bogus'"):
        config_from_json({"bogus": 1})
    with pytest.raises(ConfigError, match="unknown config key 'dataset.x'"):
        config_from_json({"dataset": {"x": 1}})
    with pytest.raises(ConfigError, match="unknown config key 'dataset.synthetic.y'"):
        config_from_json({"dataset": {"synthetic": {"y": 1}}})


@pytest.mark.parametrize("patch,msg", [
    ({"d_z": 0}, "d_z must be >= 1"), ({"epochs": 0}, "epochs must be >= 1"),
    ({"batch_size": 0}, "batch_size must be >= 1"), ({"lr": -1.0}, "lr must be >= 0"),
    ({"beta1": 1.0}, r"betas must lie in \[0, 1\)"), ({"adam_eps": 0.0}, "adam_eps must be > 0"),
    ({"bn_momentum": 2.0}, r"bn_momentum must lie in \[0, 1\]"), ({"clamp": 0.5}, r"clamp must lie in \(0, 0.5\)"),
    ({"init_std": 0.0}, "init_std must be > 0"), ({"workers": -1}, "workers must be >= 0"),
    ({"arch": "dc32"}, "unknown arch 'dc32'"), ({"out_dir": ""}, "out_dir must be non-empty"),
    ({"dataset": {"kind": "mnist"}}, "unknown dataset kind 'mnist'"),
    ({"mode": "unified-gan"}, "unknown mode 'unified-gan'"),
])
def test_validation_messages(patch, msg):
    with pytest.raises(ConfigError, match=msg):
        config_from_json(patch)


def test_valid_config_and_auto_arch():
    cfg = config_from_json({"epochs": 2, "batch_size": 16, "lr": 1e-4, "seed": 9, "out_dir": "x",
                            "dataset": {"kind": "synthetic",
                                        "synthetic": {"kind": "cosine-field", "k": 3, "per_class_n": 32,
                                                      "seed": 5, "image_size": 32}}})
    assert cfg.resolved_arch() == 2 and cfg.epochs == 2 and cfg.dataset.synthetic.k == 3


def test_cli_config_error_exits_2(tmp_path):
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"epochs": 1, "nope": 1}))
    r = subprocess.run([sys.executable, "-m", "paper_2102_10485_b200", "train", "--config", str(f)],
                       capture_output=True, text=True)
    assert r.returncode == 2 and "unknown config key 'nope'" in r.stderr


def test_estimate_priors():
    counts, probs = estimate_priors([(0, [0, 1, 2]), (1, [3])])
    assert counts.tolist() == [3, 1] and np.allclose(probs, [0.75, 0.25])
    with pytest.raises(ValueError, match="class 1 has no samples"):
        estimate_priors([(0, [0]), (1, [])])
    with pytest.raises(ValueError, match="shard class id 5 out of range"):
        estimate_priors([(5, [0])])
