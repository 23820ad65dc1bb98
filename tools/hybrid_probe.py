"""Timing probe (not a bench line) of a hybrid ResNet step at batch 256, A2W1 bipolar: the layers in
`--tcw` on the window path (one window pack + one tcw conv launch, own stream), the rest on the
expansion kernel (one grouped bit-plane pack + grouped tc convs on two streams), L2 flushed between
steps, CUDA graph.  Prints one JSON object per partition.

    python tools/hybrid_probe.py --tcw "2,5,6,8" --tc "4,7|9,10,11,12"
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

DEV = "cuda"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spec", action="append", default=[], help='"tcw=2,5,6,8;tc=4,7|9,10,11,12"')
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    layers = list(inputs.BASELINE_LAYERS)
    data = {}
    for li in layers:
        L = inputs.TABLE1[li]
        act, wt = inputs.conv_operands(L, 256, 2, 1, inputs.seed_for(3, 2, 1, "bipolar", li))
        act = act.to(DEV)
        wp = bs.bitpack(wt.reshape(L.oc * L.k * L.k, L.ic).to(DEV), 1)
        oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
        out = torch.empty((256, oh, oh, L.oc), dtype=torch.int32, device=DEV)
        w_tc = bs.conv2d_tc_prepare_weights(wp, 1, bs.BIPOLAR, L.oc, L.k, L.k, L.ic)
        packed = torch.empty((2, 256 * L.h * L.w, bs.packed_row_words(L.ic)), dtype=torch.int32, device=DEV)
        ww = bs.conv2d_tcw_prepare_weights(wp, 1, bs.BIPOLAR, L.oc, L.k, L.k, L.ic)
        aw = torch.empty(bs.tcw_act_bytes(256, L.h, L.w, L.ic, L.k, L.k, L.s, L.pad, 2), dtype=torch.uint8, device=DEV)
        data[li] = dict(L=L, act=act, out=out, tc=dict(act_packed=packed, w_tc=w_tc, out=out, n=256, h=L.h, w=L.w,
                                                            c=L.ic, oc=L.oc, kh=L.k, kw=L.k, stride=L.s, pad=L.pad,
                                                            w_enc=1),
                        packed=packed, tcw=dict(act_win=aw, w_win=ww, out=out, n=256, h=L.h, w=L.w, c=L.ic, oc=L.oc,
                                                kh=L.k, kw=L.k, stride=L.s, pad=L.pad, w_enc=1),
                        pk=dict(x=act, kh=L.k, kw=L.k, stride=L.s, pad=L.pad), aw=aw)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    specs = a.spec or ["tcw=;tc=2|4,5,6,7|8,9,10,11,12"]
    for spec in specs:
        parts = dict(x.split("=") for x in spec.split(";"))
        tcw = [int(x) for x in parts.get("tcw", "").split(",") if x]
        tcg = [[int(x) for x in g.split(",")] for g in parts.get("tc", "").split("|") if g]
        tcl = [li for g in tcg for li in g]
        s_pack, s_w, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        evp, evw = torch.cuda.Event(), torch.cuda.Event()
        mode = parts.get("mode", "")

        def step():
            main = torch.cuda.current_stream()
            for s in (s_pack, s_w, s2):
                s.wait_stream(main)
            if mode == "sp":  # packs serialized on one stream (bit planes first), each conv after its own pack
                with torch.cuda.stream(s_pack):
                    bs.bitpack_group([data[li]["act"] for li in tcl], 2, outs=[data[li]["packed"] for li in tcl])
                    evp.record(s_pack)
                    bs.digitpack_win_group([data[li]["pk"] for li in tcw], 2, outs=[data[li]["aw"] for li in tcw])
                    evw.record(s_pack)
                main.wait_event(evp)
                bs.bitserial_conv2d_nhwc_tc_group([data[li]["tc"] for g in tcg for li in g], 2, 1)
                s_w.wait_event(evw)
                with torch.cuda.stream(s_w):
                    bs.bitserial_conv2d_nhwc_tcw_group([data[li]["tcw"] for li in tcw], 2, 1)
                for s in (s_pack, s_w, s2):
                    main.wait_stream(s)
                return
            if mode == "wp":  # packs serialized, window layout first
                with torch.cuda.stream(s_pack):
                    bs.digitpack_win_group([data[li]["pk"] for li in tcw], 2, outs=[data[li]["aw"] for li in tcw])
                    evw.record(s_pack)
                    bs.bitpack_group([data[li]["act"] for li in tcl], 2, outs=[data[li]["packed"] for li in tcl])
                    evp.record(s_pack)
                s_w.wait_event(evw)
                with torch.cuda.stream(s_w):
                    bs.bitserial_conv2d_nhwc_tcw_group([data[li]["tcw"] for li in tcw], 2, 1)
                main.wait_event(evp)
                bs.bitserial_conv2d_nhwc_tc_group([data[li]["tc"] for g in tcg for li in g], 2, 1)
                for s in (s_pack, s_w, s2):
                    main.wait_stream(s)
                return
            if tcw:
                with torch.cuda.stream(s_w):
                    bs.digitpack_win_group([data[li]["pk"] for li in tcw], 2, outs=[data[li]["aw"] for li in tcw])
                    bs.bitserial_conv2d_nhwc_tcw_group([data[li]["tcw"] for li in tcw], 2, 1)
            if tcl:
                with torch.cuda.stream(s_pack):
                    bs.bitpack_group([data[li]["act"] for li in tcl], 2, outs=[data[li]["packed"] for li in tcl])
                    evp.record(s_pack)
                for gi, g in enumerate(tcg):
                    cs = (main, s2)[gi % 2]
                    cs.wait_event(evp)
                    with torch.cuda.stream(cs):
                        bs.bitserial_conv2d_nhwc_tc_group([data[li]["tc"] for li in g], 2, 1)
            for s in (s_pack, s_w, s2):
                main.wait_stream(s)
        main = torch.cuda.current_stream()
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(main)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(g, stream=cap):
                step()
        main.wait_stream(cap)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(main)
            g.replay()
            e1.record(main)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(json.dumps({"spec": spec, "median_ms": ts[len(ts) // 2], "mean_ms": sum(ts) / len(ts)}), flush=True)


if __name__ == "__main__":
    main()
