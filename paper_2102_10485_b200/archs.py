"""Layer lists of the BASELINE.json configurations c1..c4 in the text form
both the native library and the test oracle parse.

Reference conventions: every conv / transposed
conv is k4 s2 p1 with a bias; generator head FC -> Reshape -> BN -> ReLU; BN on
every discriminator conv but the first; LeakyReLU slope 0.2; BN eps 1e-5,
momentum 0.1; c2's "FC->256*4*4" is read as FC, BN, ReLU (analogy with c1).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Arch:
    name: str
    gen: str
    disc: str
    image: tuple[int, int, int]
    d_z: int = 100


def _gen(d_z: int, c0: int, side: int, chans: list[int], out_c: int) -> str:
    parts = [f"dense {d_z} {c0 * side * side}", f"reshape {c0} {side} {side}", f"bn {c0}", "relu"]
    prev = c0
    for c in chans:
        parts += [f"convT2d {prev} {c} 4 2 1", f"bn {c}", "relu"]
        prev = c
    parts += [f"convT2d {prev} {out_c} 4 2 1", "tanh"]
    return "; ".join(parts)


def _disc(in_c: int, chans: list[int], side: int) -> str:
    parts = [f"conv2d {in_c} {chans[0]} 4 2 1", "lrelu 0.2"]
    for a, b in zip(chans[:-1], chans[1:]):
        parts += [f"conv2d {a} {b} 4 2 1", f"bn {b}", "lrelu 0.2"]
    f = chans[-1] * side * side
    parts += [f"reshape {f}", f"dense {f} 1", "sigmoid"]
    return "; ".join(parts)


def baseline_arch(cfg: int, d_z: int = 100) -> Arch:
    if cfg == 1:
        return Arch("c1", _gen(d_z, 128, 7, [64], 1), _disc(1, [64, 128], 7), (1, 28, 28), d_z)
    if cfg in (2, 3):
        return Arch(f"c{cfg}", _gen(d_z, 256, 4, [128, 64], 3), _disc(3, [64, 128, 256], 4), (3, 32, 32), d_z)
    if cfg == 4:
        return Arch("c4", _gen(d_z, 512, 4, [256, 128, 64], 3), _disc(3, [64, 128, 256, 512], 4), (3, 64, 64), d_z)
    raise ValueError("config must be 1..4")


# BASELINE.json configs: (arch id, labels, images per label, per-label batch)
CONFIGS = {
    "c1": dict(arch=1, labels=10, per_label=6000, batch=64),
    "c2": dict(arch=2, labels=10, per_label=5000, batch=64),
    "c3": dict(arch=3, labels=100, per_label=500, batch=32),
    "c4": dict(arch=4, labels=1000, per_label=1280, batch=32),
    # weak-scaling sweep: 125 labels per GPU of the c4 architecture
    "sweep": dict(arch=4, labels_per_gpu=125, per_label=1280, batch=32),
}


def macs_per_image(arch: Arch) -> tuple[float, float]:
    """(generator, discriminator) forward multiply-accumulates per image."""
    def walk(spec: str, shape: tuple) -> float:
        macs = 0.0
        for item in spec.split(";"):
            tok = item.split()
            if not tok:
                continue
            if tok[0] == "dense":
                i, o = int(tok[1]), int(tok[2])
                macs += i * o
                shape = (o,)
            elif tok[0] in ("conv2d", "convT2d"):
                ci, co, k, s, p = map(int, tok[1:6])
                _, h, w = shape
                if tok[0] == "conv2d":
                    oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
                    macs += oh * ow * co * ci * k * k
                else:
                    oh, ow = (h - 1) * s - 2 * p + k, (w - 1) * s - 2 * p + k
                    macs += h * w * ci * co * k * k
                shape = (co, oh, ow)
            elif tok[0] == "reshape":
                shape = tuple(int(t) for t in tok[1:])
        return macs
    return walk(arch.gen, (arch.d_z,)), walk(arch.disc, arch.image)


def algorithmic_flops_per_image(arch: Arch) -> float:
    """2 * (4 Gf + 8 Df - 2 d1 - g1) — the minimal FLOPs of one
    full G+D step per real image (D-step: G fwd + 2 D fwd + 2x(wgrad+dgrad)
    minus the unneeded first-layer dgrad; G-step: G fwd, D fwd, D dgrad, G
    wgrad+dgrad minus the FC dgrad)."""
    gf, df = macs_per_image(arch)
    # first-layer MACs of D and G
    d1 = _first_linear_macs(arch.disc, arch.image)
    g1 = _first_linear_macs(arch.gen, (arch.d_z,))
    return 2.0 * (4 * gf + 8 * df - 2 * d1 - g1)


def _first_linear_macs(spec: str, shape: tuple) -> float:
    for item in spec.split(";"):
        tok = item.split()
        if tok and tok[0] == "dense":
            return float(int(tok[1]) * int(tok[2]))
        if tok and tok[0] == "conv2d":
            ci, co, k, s, p = map(int, tok[1:6])
            _, h, w = shape
            oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
            return float(oh * ow * co * ci * k * k)
    return 0.0


def with_bn(arch: Arch, eps: float, momentum: float) -> Arch:
    """the same architecture with explicit BatchNorm epsilon / momentum
    (RunConfig bn_eps / bn_momentum, layers.hpp:25-29)"""
    def fix(spec: str) -> str:
        out = []
        for item in spec.split(";"):
            t = item.split()
            if t and t[0] == "bn":
                item = f" bn {t[1]} {eps!r} {momentum!r}"
            out.append(item)
        return ";".join(out)
    return Arch(arch.name, fix(arch.gen), fix(arch.disc), arch.image, arch.d_z)
