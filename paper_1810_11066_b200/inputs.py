"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic: it only draws uniform integer
codes from seeded torch CPU generators and lists the workload shapes (PAPER.md
Table 1, :733-746; BASELINE.json configs).  Both the CUDA path and the oracle
consume what it returns; neither is imported here.

Recipe: codes are uniform over [0, 2^bits) for every operand —
activations unsigned, weights uniform codes (so bipolar +/-1 or +/-1/+/-3 values are
equiprobable).  Seeds follow SURVEY §8d:
    seed = 1810_11066 + 1000*config + 10*precision_id + encoding_id  (+ layer offset)
Full-size tensors are generated once on the CPU and sliced per rank, so every GPU
count sees identical data.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

BASE_SEED = 1810_11066


@dataclass(frozen=True)
class ConvLayer:
    """One row of PAPER.md Table 1 (:733-746).  `pad` is reading R4:
    1 for 3x3, 0 for 1x1 (Table 1 has no pad column; BASELINE config 1 states pad 1)."""
    name: int
    h: int
    w: int
    ic: int
    oc: int
    k: int
    s: int

    @property
    def pad(self) -> int:
        return 1 if self.k == 3 else 0


# PAPER.md:736-746 (Table 1, "Configurations of 2D-convolution operators in ResNet-18")
TABLE1 = {
    2: ConvLayer(2, 56, 56, 64, 64, 3, 1),
    3: ConvLayer(3, 56, 56, 64, 64, 1, 1),
    4: ConvLayer(4, 56, 56, 64, 128, 3, 2),
    5: ConvLayer(5, 56, 56, 64, 128, 1, 2),
    6: ConvLayer(6, 28, 28, 128, 128, 3, 1),
    7: ConvLayer(7, 28, 28, 128, 256, 3, 2),
    8: ConvLayer(8, 28, 28, 128, 256, 1, 2),
    9: ConvLayer(9, 14, 14, 256, 256, 3, 1),
    10: ConvLayer(10, 14, 14, 256, 512, 3, 2),
    11: ConvLayer(11, 14, 14, 256, 512, 1, 2),
    12: ConvLayer(12, 7, 7, 512, 512, 3, 1),
}
# BASELINE.json configs[2]/[3]: the ten body layers (Table 1 without layer 3)
BASELINE_LAYERS = (2, 4, 5, 6, 7, 8, 9, 10, 11, 12)

# (a_bits, w_bits) pairs named by BASELINE.json; id used in the seed
PRECISIONS = {(1, 1): 0, (2, 1): 1, (2, 2): 2, (1, 2): 3, (4, 1): 4, (4, 2): 5,
              (1, 3): 6, (1, 4): 7, (2, 3): 8, (2, 4): 9}
ENCODINGS = {"unipolar": 0, "bipolar": 1}


def seed_for(config: int, a_bits: int, w_bits: int, encoding: str, layer: int = 0) -> int:
    pid = PRECISIONS.get((a_bits, w_bits), 10 * a_bits + w_bits)
    return BASE_SEED + 100_000 * layer + 1000 * config + 10 * pid + ENCODINGS[encoding]


def codes(shape, bits: int, generator: torch.Generator) -> torch.Tensor:
    """Uniform codes in [0, 2^bits) as a CPU uint8 tensor."""
    return torch.randint(0, 1 << bits, tuple(shape), dtype=torch.uint8, generator=generator)


def gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def conv_operands(layer: ConvLayer, batch: int, a_bits: int, w_bits: int, seed: int):
    """(act NHWC [batch][h][w][ic], wt OHWI [oc][k][k][ic]) uint8 codes."""
    g = gen(seed)
    act = codes((batch, layer.h, layer.w, layer.ic), a_bits, g)
    wt = codes((layer.oc, layer.k, layer.k, layer.ic), w_bits, g)
    return act, wt


def dense_operands(m: int, n: int, k: int, a_bits: int, w_bits: int, seed: int):
    """(a [m][k], w [n][k]) uint8 codes."""
    g = gen(seed)
    return codes((m, k), a_bits, g), codes((n, k), w_bits, g)
