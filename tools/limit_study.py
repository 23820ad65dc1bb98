"""Limit study (Sec. 6.2.3): ResNet-18 layer 9
(14x14, 256->256, 3x3 s1, Table 1) at every A, W in 1..4, batch 1 and
batch 256, unipolar; device time of the conv kernel (events, median), binary TOPS,
and the time ratios the paper quotes ("W1A1 ... 14.4X faster than W4A4", "W2A2
1.3x better" than W1A4; paper naming WxAy = our AyWx).  Parity of every cell is
checked in tests/test_parity_gpu.py::test_limit_study_grid_parity.

    python tools/limit_study.py [--path tc|popc] > gpurun_out/limit_study.json
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402


PATH = "popc"


def time_layer(L, batch, a_bits, w_bits, reps=20):
    g = inputs.gen(1000 * a_bits + w_bits + batch)
    act = inputs.codes((batch, L.h, L.w, L.ic), a_bits, g).cuda()
    wt = inputs.codes((L.oc * 9, L.ic), w_bits, g).cuda()
    ap, wp = bs.bitpack(act, a_bits), bs.bitpack(wt, w_bits)
    out = torch.empty((batch, L.h, L.w, L.oc), dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    if PATH == "tc":  # tensor-core path (FP4 format; prepared weights, untimed)
        w_tc = bs.conv2d_tc_prepare_weights(wp, w_bits, bs.UNIPOLAR, L.oc, 3, 3, L.ic)

        def run():
            bs.bitserial_conv2d_nhwc_tc_prepared(ap, a_bits, w_tc, w_bits, batch, L.h, L.w, L.ic, L.oc, 3, 3, 1, 1,
                                                 out=out)
    else:
        def run():
            bs.bitserial_conv2d_nhwc(ap, a_bits, wp, w_bits, bs.UNIPOLAR, batch, L.h, L.w, L.ic, L.oc, 3, 3, 1, 1,
                                     out=out)
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    ops = 2 * batch * L.h * L.w * L.oc * 9 * L.ic * a_bits * w_bits
    return ms, ops / ms / 1e9


def main():
    global PATH
    ap = argparse.ArgumentParser()
    ap.add_argument("--path", choices=["tc", "popc"], default="popc")
    PATH = ap.parse_args().path
    L = inputs.TABLE1[9]
    res = {"path": PATH}
    for batch in (1, 256):
        cells = {}
        for a in range(1, 5):
            for w in range(1, 5):
                ms, tops = time_layer(L, batch, a, w)
                cells[f"A{a}W{w}"] = {"ms": ms, "binary_tops": tops}
        c = cells
        res[f"batch{batch}"] = {
            "cells": cells,
            "ratio_A4W4_over_A1W1": c["A4W4"]["ms"] / c["A1W1"]["ms"],
            "ratio_A4W1_over_A2W2": c["A4W1"]["ms"] / c["A2W2"]["ms"],
            "paper": "PAPER.md:803-804 (Cortex-A53): W1A1 14.4x faster than W4A4; W2A2 1.3x faster than W1A4",
        }
    print(json.dumps(res))


if __name__ == "__main__":
    main()
