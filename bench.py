#!/usr/bin/env python
"""bench.py — device-timed throughput of the bitserial hot path on B200.

Default workload (BASELINE.json configs[3], the multi-GPU ResNet-18 config the
north_star reports at 1/2/4/8 GPUs): the ten ResNet-18 body conv layers (PAPER.md
Table 1 without layer 3) at global batch 256, A2W1 bipolar, NHWC, sharded by batch
across ranks with no collective on the data path.  One step = for every layer, pack
the uint8 activations (timed) + bitserial conv (int32 out); weights are
packed once, untimed.  Metric: binary TOPS = sum_layers 2*M*N*K*A*W / step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet256|conv1|gemv|resnet1|gemm] ...

Prints ONE JSON line on rank 0 (the contract in DESIGN.md §6).  `--impl reference`
times the CPU oracle (the reference arm of this tier) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1810_11066_b200 import inputs  # noqa: E402

MAX_MHZ_FALLBACK = 1965.0
POPC_PER_CLK_PER_SM = 16.0   # measured, profiles/r01_int_pipe_rates.json
L2_FLUSH_BYTES = 256 << 20


# ---------------------------------------------------------------------------- setup
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, local, backend):
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": MAX_MHZ_FALLBACK}, "fallback"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index, period=0.01):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period, self._stop = period, threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:  # noqa: BLE001 — clocks are reported as unavailable
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------ workloads
class ConvLayerRun:
    """One conv layer on this rank's batch shard: resident inputs/outputs in HBM."""

    def __init__(self, L, act_cpu, wt_cpu, a_bits, w_bits, bipolar, dev):
        import paper_1810_11066_b200 as bs
        self.bs, self.L = bs, L
        self.a_bits, self.w_bits, self.enc = a_bits, w_bits, (bs.BIPOLAR if bipolar else bs.UNIPOLAR)
        self.n = act_cpu.shape[0]
        self.act = act_cpu.to(dev)
        self.wp = bs.bitpack(wt_cpu.reshape(L.oc * L.k * L.k, L.ic).to(dev), w_bits)  # untimed
        self.oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
        self.out = torch.empty((self.n, self.oh, self.oh, L.oc), dtype=torch.int32, device=dev)
        self.ws = torch.empty(bs.conv2d_workspace_bytes(self.n, L.h, L.w, L.ic, a_bits), dtype=torch.uint8, device=dev)
        self.packed = self.ws.view(torch.int32).view(a_bits, self.n * L.h * L.w, bs.packed_row_words(L.ic))

    def binops(self, n=None):
        n = self.n if n is None else n
        L = self.L
        return 2 * n * self.oh * self.oh * L.oc * L.k * L.k * L.ic * self.a_bits * self.w_bits

    def step(self):  # pack + conv (timed unit)
        L = self.L
        self.bs.bitserial_conv2d_nhwc_i8(self.act, self.a_bits, self.wp, self.w_bits, self.enc, L.oc, L.k, L.k,
                                         L.s, L.pad, out=self.out, workspace=self.ws)

    def pack_only(self):
        self.bs.bitpack(self.act, self.a_bits, out=self.packed)

    def conv_only(self):
        L = self.L
        self.bs.bitserial_conv2d_nhwc(self.packed, self.a_bits, self.wp, self.w_bits, self.enc, self.n, L.h, L.w,
                                      L.ic, L.oc, L.k, L.k, L.s, L.pad, out=self.out)


def build_resnet(args, rank, world, dev, batch):
    lo, hi = inputs.shard_range(batch, rank, world)
    enc = "bipolar" if args.bipolar else "unipolar"
    runs = []
    for li in inputs.BASELINE_LAYERS:
        L = inputs.TABLE1[li]
        act, wt = inputs.conv_operands(L, batch, args.a_bits, args.w_bits,
                                       inputs.seed_for(4 if batch > 1 else 3, args.a_bits, args.w_bits, enc, li))
        runs.append(ConvLayerRun(L, act[lo:hi].contiguous(), wt, args.a_bits, args.w_bits, args.bipolar, dev))
    return runs, (lo, hi)


# --------------------------------------------------------------------------- timing
def time_steps(step_fn, steps, warmup, world, dev, flush=None, use_graph=True):
    """W untimed warm-ups, then K steps each bracketed by CUDA events on the launching
    stream (L2 flushed between steps, outside the events); barrier + synchronize on
    both sides; returns max-over-ranks mean ms/step."""
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        step_fn()
    torch.cuda.synchronize()
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                step_fn()
        stream.wait_stream(s)
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else step_fn
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier(world)
    torch.cuda.synchronize()
    for e0, e1 in ev:
        if flush is not None:
            flush.zero_()
        e0.record(stream)
        run()
        e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / steps
    return allreduce_max(ms, world, dev), graph is not None


def kernel_durations(runs, reps, world, dev):
    """Per-launch device time of the pack and conv kernels, eager, events on the
    launching stream around each launch (the roofline's denominator)."""
    stream = torch.cuda.current_stream()
    pack_ms, conv_ms = [0.0] * len(runs), [0.0] * len(runs)
    for i, r in enumerate(runs):
        r.pack_only()
        r.conv_only()
    torch.cuda.synchronize()
    for _ in range(reps):
        for i, r in enumerate(runs):
            a0, a1, b1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a0.record(stream)
            r.pack_only()
            a1.record(stream)
            r.conv_only()
            b1.record(stream)
            torch.cuda.synchronize()
            pack_ms[i] += a0.elapsed_time(a1) / reps
            conv_ms[i] += a1.elapsed_time(b1) / reps
    return pack_ms, conv_ms


def e2e_resnet(runs, steps, world, dev):
    """Same metric through the host-buffer C-ABI entry (bs_bitserial_conv2d_nhwc_host):
    H2D of pinned uint8 activations, pack, conv, D2H of the int32 outputs, per layer."""
    import paper_1810_11066_b200 as bs
    host = []
    for r in runs:
        host.append((r.act.cpu().pin_memory(), torch.empty(r.out.shape, dtype=torch.int32).pin_memory(),
                     torch.empty_like(r.act), torch.empty_like(r.out)))
    stream = torch.cuda.current_stream()

    def step():
        for r, (ah, oh_, ad, od) in zip(runs, host):
            L = r.L
            bs.bitserial_conv2d_nhwc_host(ah, r.a_bits, r.wp, r.w_bits, r.enc, L.oc, L.k, L.k, L.s, L.pad,
                                          oh_, ad, od, r.ws)
    step()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = allreduce_max(e0.elapsed_time(e1) / steps, world, dev)
    h2d = sum(h[0].numel() for h in host)
    d2h = sum(h[1].numel() * 4 for h in host)
    return ms, h2d, d2h


# ------------------------------------------------------------------------ reference
def oracle_resnet_sample(args, images):
    """CPU oracle on `images` images of the ten layers (same seeds as the GPU arm)."""
    import oracle
    enc = "bipolar" if args.bipolar else "unipolar"
    total_ops, t = 0, 0.0
    for li in inputs.BASELINE_LAYERS:
        L = inputs.TABLE1[li]
        g = inputs.gen(inputs.seed_for(4, args.a_bits, args.w_bits, enc, li))
        act = inputs.codes((images, L.h, L.w, L.ic), args.a_bits, g).numpy()
        wt = inputs.codes((L.oc, L.k, L.k, L.ic), args.w_bits, g).numpy()
        t0 = time.perf_counter()
        oracle.conv2d_nhwc(act, args.a_bits, wt, args.w_bits, args.bipolar, stride=(L.s, L.s), pad=(L.pad, L.pad))
        t += time.perf_counter() - t0
        oh = (L.h + 2 * L.pad - L.k) // L.s + 1
        total_ops += 2 * images * oh * oh * L.oc * L.k * L.k * L.ic * args.a_bits * args.w_bits
    return total_ops, t


def cpu_baseline(args, budget_s=15.0):
    import oracle
    ops1, t1 = oracle_resnet_sample(args, 1)
    imgs = max(1, min(16, int(budget_s / max(t1, 1e-3))))
    if imgs > 1:
        ops, t = oracle_resnet_sample(args, imgs)
    else:
        ops, t = ops1, t1
    return {"value": ops / t / 1e12, "unit": "binary TOPS", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{imgs} image(s) of the 10 ResNet-18 layers (batch-256 seeds, images 0..{imgs - 1}), "
                      f"A{args.a_bits}W{args.w_bits} {'bipolar' if args.bipolar else 'unipolar'}, OpenMP C oracle",
            "seconds": t}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_resnet_sample(args, 1)
    ts, ops = [], 0
    for _ in range(args.steps):
        ops, t = oracle_resnet_sample(args, 1)
        ts.append(t)
    ms = 1e3 * sum(ts) / len(ts)
    value = ops / (ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "binary TOPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8->i32", "data": "synthetic (seeded uniform codes)", "impl": "reference",
        "config": {"workload": "resnet18_layers2-12_b256_a2w1_bipolar", "sample_per_step": "1 image of the 10 layers",
                   "a_bits": args.a_bits, "w_bits": args.w_bits},
        "cpu_baseline": {"value": value, "unit": "binary TOPS", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": "1 image of the 10 ResNet-18 layers per step (the batch-256 workload's images "
                                   "are independent; the oracle runs a bounded sample)"},
        "e2e": {"value": value, "unit": "binary TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


METRIC = "bitserial conv/GEMM binary TOPS (device-timed) and % of int-pipe/HBM roofline"


# ---------------------------------------------------------------------------- main
def run_ours(args):
    world, rank, local = dist_env()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    init_dist(world, local, "nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1810_11066_b200 as bs
    bs._load()
    peaks, peaks_src = measured_peaks()
    batch = 256
    runs, (lo, hi) = build_resnet(args, rank, world, dev, batch)
    step = lambda: [r.step() for r in runs]  # noqa: E731
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    # launches per step, counted by the library itself on one eager step
    n0 = bs.kernel_launches()
    step()
    torch.cuda.synchronize()
    launches_per_step = bs.kernel_launches() - n0

    with ClockSampler(local) as clk:
        ms, graphed = time_steps(step, args.steps, args.warmup, world, dev, flush=flush, use_graph=not args.no_graph)
    clocks = clk.summary()

    total_binops = sum(r.binops(batch) for r in runs)  # whole job: global batch
    value = total_binops / (ms / 1e3) / 1e12

    # roofline of the dominant kernel (the conv kernel): algorithmic binary ops / its
    # own device time, against the integer-pipe bound R_int: per 32-bit
    # word pair one LOP3 (AND) on the ALU (64/clk/SM) plus counting, either one POPC on
    # the XU (16/clk/SM) or a carry-save full adder (2 LOP3); balancing the two pipes
    # gives 32 word pairs/clk/SM = 2 x R_popc (R_popc: one POPC per word pair).
    pack_ms, conv_ms = kernel_durations(runs, max(3, min(args.steps, 10)), world, dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_max = (clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz") or MAX_MHZ_FALLBACK)
    r_popc = 64.0 * POPC_PER_CLK_PER_SM * sms * f_max * 1e6 / 1e12
    r_int = 2.0 * r_popc
    conv_total_ms = sum(conv_ms)
    rank_binops = sum(r.binops() for r in runs)
    achieved = rank_binops / (conv_total_ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r01_conv_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("dram_bytes_per_step")
    pack_bytes = sum(r.act.numel() * (1 + r.a_bits / 8) for r in runs)
    pack_gbs = pack_bytes / (sum(pack_ms) / 1e3) / 1e9

    e2e = None
    if not args.no_e2e:
        ems, h2d, d2h = e2e_resnet(runs, max(1, min(args.steps, 5)), world, dev)
        e2e = {"value": total_binops / (ems / 1e3) / 1e12, "unit": "binary TOPS",
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world, "ms_per_step": ems}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "binary TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8->i32 (AND/POPC on packed u32 bit-planes)",
            "data": "synthetic (seeded uniform codes, PAPER.md Table 1 shapes; no dataset)",
            "config": {
                "workload": f"resnet18_layers2-12_b{batch}_a{args.a_bits}w{args.w_bits}_"
                            f"{'bipolar' if args.bipolar else 'unipolar'}",
                "global_batch": batch, "layers": list(inputs.BASELINE_LAYERS), "layout": "NHWC/OHWI",
                "parallelism": f"batch-sharded dp{world} (no collective)", "rank0_images": [lo, hi],
                "step": "per layer: bitpack(act) + bitserial conv2d (weights prepacked, untimed)",
                "l2": "256 MiB buffer zeroed between timed steps (outside the events)", "cuda_graph": graphed,
            },
            "roofline": {"bound": "alu", "achieved": achieved, "peak": r_int, "unit": "binary TOPS",
                         "frac": achieved / r_int, "traffic": traffic, "r_popc": r_popc,
                         "frac_r_popc": achieved / r_popc,
                         "kernel": "popc_conv_kernel (sum over the 10 layer launches of one step, rank 0)",
                         "peak_basis": f"integer pipes (measured rates, profiles/r01_int_pipe_rates.json): per "
                                       f"32-bit word pair 1 LOP3 + {{1 POPC | 2 LOP3}} balanced -> 32 word pairs/"
                                       f"clk/SM x 64 binary ops x {sms} SMs x {f_max:.0f} MHz (= 2 x R_popc)"},
            "breakdown": {"conv_ms": conv_ms, "pack_ms": pack_ms, "pack_gbs": pack_gbs,
                          "pack_frac_hbm": pack_gbs / peaks["hbm_gbs"], "hbm_peak_gbs": peaks["hbm_gbs"],
                          "peaks_source": peaks_src},
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "launches_per_step": launches_per_step,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--a-bits", type=int, default=2)
    ap.add_argument("--w-bits", type=int, default=1)
    ap.add_argument("--unipolar", dest="bipolar", action="store_false")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
