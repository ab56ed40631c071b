"""The five BASELINE.json workloads (configs[0..4]) and their reduced parity sizes.

Each entry: the generator spec (inputs.generate.GenSpec), k, l, the priming and
its hyper-parameters, the row layout used when sharding over GPUs.  Seeds follow
SURVEY.md §8(d): data seed 1000 + index, init seed 2000 + index.
"""
from __future__ import annotations

import dataclasses

from .generate import GenSpec


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    spec: GenSpec
    k: int
    l: int
    priming: str               # 'power' | 'oja' | 'eigengame'
    iters: int = 0             # power iterations
    batch: int = 0             # minibatch rows (oja / eigengame)
    alpha: float = 0.0
    momentum: float = 0.9      # Nesterov factor, §5
    steps: int = 0             # default minibatch step budget for tests/bench
    init_seed: int = 0
    layout: str = "contiguous"

    @property
    def m(self) -> int:
        return self.k + self.l


C1 = Workload("C1", GenSpec("planted_qr", n=2000, d=64, seed=1000, spectrum="exp", a=4.0),
              k=4, l=4, priming="power", iters=20, init_seed=2000)
C2 = Workload("C2", GenSpec("image_factor", n=60000, d=784, seed=1001),
              k=16, l=16, priming="oja", batch=256, alpha=1e-3, steps=2350, init_seed=2001,
              layout="interleaved")
C3 = Workload("C3", GenSpec("planted_qr", n=1_000_000, d=1024, seed=1002, spectrum="exp", a=20.0),
              k=32, l=32, priming="power", iters=50, init_seed=2002)
C4 = Workload("C4", GenSpec("planted_qr", n=2_000_000, d=4096, seed=1003, spectrum="power", a=1.5, noise=1e-4),
              k=32, l=32, priming="eigengame", batch=4096, alpha=1e-4, steps=489, init_seed=2003,
              layout="interleaved")
C5 = Workload("C5", GenSpec("planted_householder", n=200_000, d=65536, seed=1004, spectrum="power", a=1.0,
                            relu=True, house_r=8, dtype="bf16"),
              k=64, l=64, priming="power", iters=30, init_seed=2004)

FULL = {w.name: w for w in (C1, C2, C3, C4, C5)}

# Reduced sizes with the same family/spectrum/priming: the oracle finishes them in seconds and
# they still span several row tiles and a ragged tail (n not a multiple of any tile or batch).
SMALL = {
    "C1": C1,
    "C2s": dataclasses.replace(C2, name="C2s", spec=dataclasses.replace(C2.spec, n=12_096), steps=200),
    "C3s": dataclasses.replace(C3, name="C3s", spec=dataclasses.replace(C3.spec, n=100_003, d=256), iters=12),
    "C4s": dataclasses.replace(C4, name="C4s", spec=dataclasses.replace(C4.spec, n=41_216, d=512),
                               batch=4096, steps=30),
    "C5s": dataclasses.replace(C5, name="C5s", spec=dataclasses.replace(C5.spec, n=6_007, d=2048), iters=8),
}
