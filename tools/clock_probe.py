"""SM clock and throttle reasons while one tensor-core conv layer (batch 256) is replayed
back to back for ~1 s in a CUDA graph: does the FP4 MMA load pull the clock below max?
Usage: python tools/clock_probe.py [--layers 6,12,2] [--a 2 --w 1] [--fmt f4|i8]"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="6,12,2")
ap.add_argument("--a", type=int, default=2)
ap.add_argument("--w", type=int, default=1)
ap.add_argument("--fmt", default="f4")
ap.add_argument("--seconds", type=float, default=1.0)
args = ap.parse_args()
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
fmt = bs.TC_F4 if args.fmt == "f4" else bs.TC_I8
dev = torch.device("cuda")
for li in map(int, args.layers.split(",")):
    L = inputs.TABLE1[li]
    g = inputs.gen(li)
    act = inputs.codes((256, L.h, L.w, L.ic), args.a, g).to(dev)
    wt = inputs.codes((L.oc * L.k * L.k, L.ic), args.w, g).to(dev)
    ap_ = bs.bitpack(act, args.a)
    w_tc = bs.conv2d_tc_prepare_weights(bs.bitpack(wt, args.w), args.w, bs.BIPOLAR, L.oc, L.k, L.k, L.ic, tc_format=fmt)
    oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
    out = torch.empty((256, oh, oh, L.oc), dtype=torch.int32, device=dev)
    run = lambda: bs.bitserial_conv2d_nhwc_tc_prepared(ap_, args.a, w_tc, args.w, 256, L.h, L.w, L.ic, L.oc,  # noqa
                                                       L.k, L.k, L.s, L.pad, out=out, tc_format=fmt)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        run()
        s.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(50):
                run()
    samples, reasons, stop = [], set(), threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            for bit, name in ((0x4, "sw_power_cap"), (0x8, "hw_slowdown"), (0x20, "sw_thermal"), (0x40, "hw_thermal")):
                if r & bit:
                    reasons.add(name)
            time.sleep(0.002)
    with torch.cuda.stream(s):
        gr.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = threading.Thread(target=sampler)
        t.start()
        n = 0
        e0.record(s)
        t0 = time.time()
        while time.time() - t0 < args.seconds:
            gr.replay()
            n += 1
            if n % 4 == 0:
                s.synchronize()
        e1.record(s)
        s.synchronize()
        stop.set()
        t.join()
    us = e0.elapsed_time(e1) * 1e3 / (50 * n)
    print(json.dumps({"layer": li, "a": args.a, "w": args.w, "fmt": args.fmt, "us_per_launch": round(us, 2),
                      "sm_mhz_median": statistics.median(samples), "sm_mhz_min": min(samples),
                      "power_w": pynvml.nvmlDeviceGetPowerUsage(h) / 1e3, "reasons": sorted(reasons),
                      "samples": len(samples)}))
