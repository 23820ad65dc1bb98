"""Timing probe of the window path (not a bench line): per-layer and grouped tcw conv launches
of the ResNet-18 body at batch 256 (A2W1 bipolar), the grouped window pack, and a step-like
sequence (pack group + conv groups, L2 flush between steps).  Each launch timed in a CUDA graph
of `reps` copies with events on the replaying stream.  Prints one JSON object.

    python tools/tcw_probe.py [--reps 20] [--layers] [--groups "all;2,4,5,6,7|8,9,10,11,12"]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402
from bench import graph_launch_ms, measured_peaks  # noqa: E402

DEV = "cuda"


def setup(batch, a_bits, w_bits, layers):
    runs = []
    for li in layers:
        L = inputs.TABLE1[li]
        act, wt = inputs.conv_operands(L, batch, a_bits, w_bits, inputs.seed_for(3, a_bits, w_bits, "bipolar", li))
        act = act.to(DEV)
        wp = bs.bitpack(wt.reshape(L.oc * L.k * L.k, L.ic).to(DEV), w_bits)
        ww = bs.conv2d_tcw_prepare_weights(wp, w_bits, bs.BIPOLAR, L.oc, L.k, L.k, L.ic)
        aw = torch.empty(bs.tcw_act_bytes(batch, L.h, L.w, L.ic, L.k, L.k, L.s, L.pad, a_bits), dtype=torch.uint8,
                         device=DEV)
        oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
        out = torch.empty((batch, oh, oh, L.oc), dtype=torch.int32, device=DEV)
        runs.append(dict(L=L, act=act, aw=aw, pk=dict(x=act, kh=L.k, kw=L.k, stride=L.s, pad=L.pad),
                         item=dict(act_win=aw, w_win=ww, out=out, n=batch, h=L.h, w=L.w, c=L.ic, oc=L.oc, kh=L.k,
                                   kw=L.k, stride=L.s, pad=L.pad, w_enc=1),
                         out_bytes=out.numel() * 4, in_bytes=aw.numel() + ww.numel()))
    return runs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--layers", action="store_true")
    ap.add_argument("--groups", default="all;2,4,5,6,7|8,9,10,11,12;2|4,5,6,7,8,9,10,11,12")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--a", type=int, default=2)
    ap.add_argument("--w", type=int, default=1)
    a = ap.parse_args()
    peaks = measured_peaks()[0]
    hbm = peaks["hbm_gbs"]
    res = {"hbm_peak_gbs": hbm, "a": a.a, "w": a.w, "batch": a.batch}
    layers = list(inputs.BASELINE_LAYERS)
    runs = setup(a.batch, a.a, a.w, layers)
    pack = lambda: bs.digitpack_win_group([r["pk"] for r in runs], a.a, outs=[r["aw"] for r in runs])  # noqa: E731
    pack()
    torch.cuda.synchronize()
    pms = graph_launch_ms(pack, a.reps)
    pbytes = sum(r["act"].numel() + r["aw"].numel() for r in runs)
    res["pack_group_us"] = 1e3 * pms
    res["pack_group_gbs"] = pbytes / pms / 1e6
    if a.layers:
        per = []
        for r in runs:
            f = lambda r=r: bs.bitserial_conv2d_nhwc_tcw_group([r["item"]], a.a, a.w)  # noqa: E731
            ms = graph_launch_ms(f, a.reps)
            per.append({"layer": r["L"].name, "us": 1e3 * ms, "out_gbs": r["out_bytes"] / ms / 1e6,
                        "t_out_us_at_peak": r["out_bytes"] / hbm / 1e3})
        res["layers"] = per
        res["layers_sum_us"] = sum(p["us"] for p in per)
    tot_bytes = sum(r["out_bytes"] + r["in_bytes"] for r in runs)
    for spec in a.groups.split(";"):
        parts = [layers] if spec == "all" else [[int(x) for x in p.split(",")] for p in spec.split("|")]
        fns = [lambda p=p: bs.bitserial_conv2d_nhwc_tcw_group([runs[layers.index(li)]["item"] for li in p], a.a, a.w)
               for p in parts]
        gms = [graph_launch_ms(f, a.reps) for f in fns]
        res[f"groups {spec}"] = {"us": [1e3 * t for t in gms], "sum_us": 1e3 * sum(gms),
                                 "hbm_frac": tot_bytes / (sum(gms) / 1e3) / 1e9 / hbm}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    for spec in a.groups.split(";"):
        parts = [layers] if spec == "all" else [[int(x) for x in p.split(",")] for p in spec.split("|")]
        s2 = torch.cuda.Stream()

        def step():
            main_s = torch.cuda.current_stream()
            pack()
            s2.wait_stream(main_s)
            streams = [main_s, s2]
            for gi, p in enumerate(parts):
                with torch.cuda.stream(streams[gi % 2]):
                    bs.bitserial_conv2d_nhwc_tcw_group([runs[layers.index(li)]["item"] for li in p], a.a, a.w)
            main_s.wait_stream(s2)
        main_s = torch.cuda.current_stream()
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(main_s)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap):
                step()
        main_s.wait_stream(cap)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main_s)
            g.replay()
            e1.record(main_s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res[f"step {spec}"] = {"median_ms": ts[len(ts) // 2], "mean_ms": sum(ts) / len(ts)}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
