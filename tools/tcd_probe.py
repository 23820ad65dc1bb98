"""Timing probe of the digit-packed TMA-fed tensor-core path (not a bench line): per-layer and
grouped conv launches of the ResNet-18 body at batch 256 (A2W1 bipolar), the grouped digit
pack, a step-like sequence (pack group + conv groups on two streams, with an L2 flush
between steps), and the GEMM sweep shapes.  Each launch timed in a CUDA graph of `reps`
copies with events on the replaying stream.  Prints one JSON object.

    python tools/tcd_probe.py [--reps 20] [--gemm] [--layers]
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


def conv_setup(batch, a_bits, w_bits, layers):
    runs = []
    for li in layers:
        L = inputs.TABLE1[li]
        act, wt = inputs.conv_operands(L, batch, a_bits, w_bits, inputs.seed_for(3, a_bits, w_bits, "bipolar", li))
        act = act.to(DEV)
        wp = bs.bitpack(wt.reshape(L.oc * L.k * L.k, L.ic).to(DEV), w_bits)
        wd = bs.conv2d_tcd_prepare_weights(wp, w_bits, bs.BIPOLAR, L.oc, L.k, L.k, L.ic)
        ad = torch.empty(((a_bits + 1) // 2, batch * L.h * L.w, bs.digit_row_bytes(L.ic)), dtype=torch.uint8,
                         device=DEV)
        oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
        out = torch.empty((batch, oh, oh, L.oc), dtype=torch.int32, device=DEV)
        runs.append(dict(L=L, act=act, ad=ad, item=dict(act_dig=ad, w_dig=wd, out=out, n=batch, h=L.h, w=L.w, c=L.ic,
                                                          oc=L.oc, kh=L.k, kw=L.k, stride=L.s, pad=L.pad, w_enc=1),
                         out_bytes=out.numel() * 4, in_bytes=ad.numel() + wd.numel()))
    return runs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--gemm", action="store_true")
    ap.add_argument("--layers", action="store_true")
    ap.add_argument("--groups", default="2|4,5,6,7,8,9,10,11,12;2,4,5,6,7|8,9,10,11,12;all")
    ap.add_argument("--epi", choices=["tma", "direct"], default="tma")
    ap.add_argument("--asrc", type=int, default=0, help="BS_TUNE_TCD_A_SRC (1 TMA im2col, 2 cp.async)")
    ap.add_argument("--bstream", type=int, default=0, help="BS_TUNE_TCD_B_STREAM")
    ap.add_argument("--batch", type=int, default=256)
    a = ap.parse_args()
    bs.set_tuning(bs.TUNE_TCD_A_SRC, a.asrc)
    bs.set_tuning(bs.TUNE_TCD_B_STREAM, a.bstream)
    if a.epi == "direct":
        bs.set_tuning(bs.TUNE_TC_EPILOGUE, 1)
    peaks = measured_peaks()[0]
    hbm = peaks["hbm_gbs"]
    res = {"hbm_peak_gbs": hbm}
    layers = list(inputs.BASELINE_LAYERS)
    runs = conv_setup(a.batch, 2, 1, layers)
    pack = lambda: bs.digitpack_group([r["act"] for r in runs], 2, outs=[r["ad"] for r in runs])  # noqa: E731
    pack()
    torch.cuda.synchronize()
    pms = graph_launch_ms(pack, a.reps)
    pbytes = sum(r["act"].numel() + r["ad"].numel() for r in runs)
    res["pack_group_us"] = 1e3 * pms
    res["pack_group_gbs"] = pbytes / pms / 1e6
    if a.layers:
        per = []
        for r in runs:
            f = lambda r=r: bs.bitserial_conv2d_nhwc_tcd_group([r["item"]], 2, 1)  # noqa: E731
            ms = graph_launch_ms(f, a.reps)
            per.append({"layer": r["L"].name, "us": 1e3 * ms, "out_gbs": r["out_bytes"] / ms / 1e6,
                        "t_out_us_at_peak": r["out_bytes"] / hbm / 1e3})
        res["layers"] = per
        res["layers_sum_us"] = sum(p["us"] for p in per)
    for spec in a.groups.split(";"):
        parts = [layers] if spec == "all" else [[int(x) for x in p.split(",")] for p in spec.split("|")]
        fns = [lambda p=p: bs.bitserial_conv2d_nhwc_tcd_group([runs[layers.index(li)]["item"] for li in p], 2, 1)
               for p in parts]
        gms = [graph_launch_ms(f, a.reps) for f in fns]
        tot_bytes = sum(r["out_bytes"] + r["in_bytes"] for r in runs)
        res[f"groups {spec}"] = {"us": [1e3 * t for t in gms], "sum_us": 1e3 * sum(gms),
                                 "hbm_frac": tot_bytes / (sum(gms) / 1e3) / 1e9 / hbm}
    # step-like: pack on a side stream, groups on two streams; L2 flush between steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    for spec in a.groups.split(";"):
        parts = [layers] if spec == "all" else [[int(x) for x in p.split(",")] for p in spec.split("|")]
        side, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        evp = torch.cuda.Event()

        def step():
            main_s = torch.cuda.current_stream()
            side.wait_stream(main_s)
            with torch.cuda.stream(side):
                pack()
                evp.record(side)
            streams = [main_s, s2]
            s2.wait_stream(main_s)
            for gi, p in enumerate(parts):
                cs = streams[gi % 2]
                cs.wait_event(evp)
                with torch.cuda.stream(cs):
                    bs.bitserial_conv2d_nhwc_tcd_group([runs[layers.index(li)]["item"] for li in p], 2, 1)
            main_s.wait_stream(s2)
            main_s.wait_stream(side)
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
    if a.gemm:
        gem = []
        for size, ab, wb in ((4096, 1, 1), (4096, 2, 1), (8192, 1, 1), (8192, 2, 1), (8192, 4, 2), (16384, 2, 1)):
            g_ = inputs.gen(size + ab)
            A = inputs.codes((size, size), ab, g_).to(DEV)
            W = inputs.codes((size, size), wb, g_).to(DEV)
            ad = bs.digitpack(A, ab)
            wd = bs.dense_tcd_prepare_weights(bs.bitpack(W, wb), wb, bs.BIPOLAR, size, size)
            out = torch.empty((size, size), dtype=torch.int32, device=DEV)
            f = lambda: bs.bitserial_dense_tcd(ad, ab, wd, wb, size, size, size, out=out, w_enc=1)  # noqa: E731
            ms = graph_launch_ms(f, max(2, a.reps // 4))
            pk = lambda: bs.digitpack(A, ab, out=ad)  # noqa: E731
            pms = graph_launch_ms(pk, max(2, a.reps // 4))
            mma_ops = 2 * size ** 3 * ((ab + 1) // 2) * ((wb + 1) // 2)
            gem.append({"size": size, "a": ab, "w": wb, "gemm_ms": ms, "pack_ms": pms,
                        "tensor_frac_fp4": mma_ops / ms / 1e9 / (4 * peaks["bf16_tflops"]),
                        "binary_tops": 2 * size ** 3 * ab * wb / (ms + pms) / 1e9})
            del A, W, ad, wd, out
        res["gemm"] = gem
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
