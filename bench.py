#!/usr/bin/env python
"""bench.py — device-timed throughput of the bitserial hot path on B200.

Default workload (BASELINE.json configs[3], the ResNet-18 config the north_star
reports at 1/2/4/8 GPUs): the ten ResNet-18 body conv layers (Table 1
without layer 3) at global batch 256, A2W1 bipolar, NHWC, sharded by batch across
ranks with no collective on the data path.  One step = for every layer, pack the
uint8 activations (timed) + bitserial conv (int32 out); weights are
packed once, untimed.  Metric: binary TOPS = sum_layers 2*M*N*K*A*W / step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet256|conv1|gemv|resnet1|gemm] [--size S]
                    [--a-bits A] [--w-bits W] [--unipolar]

Other workloads (the remaining BASELINE configs, for measurement; the driver uses
the default): conv1 = configs[0], gemv = configs[1], resnet1 = configs[2] (one
precision per run), gemm = configs[4] (row-sharded, NCCL all-gather of the int32 C).

Prints ONE JSON line on rank 0 (contract in DESIGN.md §6).  `--impl reference` times
the CPU oracle (this tier's reference arm) on the host cores instead.
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

from paper_1810_11066_b200 import dist as bsdist  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

METRIC = "bitserial conv/GEMM binary TOPS (device-timed) and % of int-pipe/HBM roofline"
MAX_MHZ_FALLBACK = 1965.0
POPC_PER_CLK_PER_SM = 16.0   # measured, profiles/r01_int_pipe_rates.json
L2_FLUSH_BYTES = 256 << 20


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": MAX_MHZ_FALLBACK}, \
            "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + clock-event (throttle) reasons during the timed region."""

    REASONS = {
        0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index, period=0.005):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period, self._stop = period, threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:  # noqa: BLE001 — reported as unavailable
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
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


def ev():
    return torch.cuda.Event(enable_timing=True)


def tc_fmt(args):
    import paper_1810_11066_b200 as bs
    return bs.TC_I8 if args.tc_format == "i8" else bs.TC_F4


def binops_conv(L, n, a_bits, w_bits):
    oh = (L.h + 2 * L.pad - L.k) // L.s + 1
    return 2 * n * oh * oh * L.oc * L.k * L.k * L.ic * a_bits * w_bits


# ----------------------------------------------------------------------- conv layers
class ConvLayerRun:
    """One conv layer on this rank's batch shard: resident inputs/outputs in HBM."""

    def __init__(self, L, act_cpu, wt_cpu, a_bits, w_bits, bipolar, dev, path="tc", fmt=0):
        import paper_1810_11066_b200 as bs
        self.bs, self.L, self.path = bs, L, path
        self.a_bits, self.w_bits, self.enc = a_bits, w_bits, (bs.BIPOLAR if bipolar else bs.UNIPOLAR)
        self.n = act_cpu.shape[0]
        self.act_cpu, self.wt_cpu = act_cpu, wt_cpu
        self.act = act_cpu.to(dev)
        self.wp = bs.bitpack(wt_cpu.reshape(L.oc * L.k * L.k, L.ic).to(dev), w_bits)  # untimed
        self.oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
        self.out = torch.empty((self.n, self.oh, self.oh, L.oc), dtype=torch.int32, device=dev)
        self.ws = torch.empty(bs.conv2d_workspace_bytes(self.n, L.h, L.w, L.ic, a_bits), dtype=torch.uint8, device=dev)
        self.packed = self.ws.view(torch.int32).view(a_bits, self.n * L.h * L.w, bs.packed_row_words(L.ic))
        # tensor-core path: weight planes expanded once, offline like the packing itself
        self.fmt = fmt
        self.w_tc = (bs.conv2d_tc_prepare_weights(self.wp, w_bits, self.enc, L.oc, L.k, L.k, L.ic, tc_format=fmt)
                     if path == "tc" else None)
        # digit path: weight digits (offline) and the digit-packed activation buffer
        self.w_dig = (bs.conv2d_tcd_prepare_weights(self.wp, w_bits, self.enc, L.oc, L.k, L.k, L.ic)
                      if path == "tcd" else None)
        self.dig = (torch.empty(((a_bits + 1) // 2, self.n * L.h * L.w, bs.digit_row_bytes(L.ic)), dtype=torch.uint8,
                                device=dev) if path == "tcd" else None)
        # window path: window-path weight digits (offline) and the window-layout activation buffer
        self.w_win = (bs.conv2d_tcw_prepare_weights(self.wp, w_bits, self.enc, L.oc, L.k, L.k, L.ic)
                      if path == "tcw" else None)
        self.win = (torch.empty(bs.tcw_act_bytes(self.n, L.h, L.w, L.ic, L.k, L.k, L.s, L.pad, a_bits),
                                dtype=torch.uint8, device=dev) if path == "tcw" else None)

    def binops(self):
        return binops_conv(self.L, self.n, self.a_bits, self.w_bits)

    def step(self):  # pack + conv (the timed unit)
        L = self.L
        if self.path == "tc":
            self.bs.bitserial_conv2d_nhwc_tc_i8(self.act, self.a_bits, self.w_tc, self.w_bits, L.oc, L.k, L.k,
                                                L.s, L.pad, out=self.out, workspace=self.ws, tc_format=self.fmt)
        else:  # --path popc: the integer-pipe kernel by name (BS_ALGO_AUTO would take the tensor cores)
            self.bs.bitpack(self.act, self.a_bits, out=self.packed)
            self.conv_only()

    def pack_only(self, max_ctas=0):
        self.bs.bitpack(self.act, self.a_bits, out=self.packed, max_ctas=max_ctas)

    def conv_only(self):
        L = self.L
        if self.path == "tc":
            self.bs.bitserial_conv2d_nhwc_tc_prepared(self.packed, self.a_bits, self.w_tc, self.w_bits, self.n, L.h,
                                                      L.w, L.ic, L.oc, L.k, L.k, L.s, L.pad, out=self.out,
                                                      tc_format=self.fmt)
        else:
            self.bs.bitserial_conv2d_nhwc(self.packed, self.a_bits, self.wp, self.w_bits, self.enc, self.n, L.h,
                                          L.w, L.ic, L.oc, L.k, L.k, L.s, L.pad, out=self.out,
                                          algo=self.bs.ALGO_POPC)

    def tcd_item(self):
        L = self.L
        return dict(act_dig=self.dig, w_dig=self.w_dig, out=self.out, n=self.n, h=L.h, w=L.w, c=L.ic, oc=L.oc,
                    kh=L.k, kw=L.k, stride=L.s, pad=L.pad, w_enc=self.enc)

    def packed_bytes(self):
        """Algorithmic activation bytes of this layer's conv: its input bit-packed (A bit planes of
        packed_row_words(c) words per pixel) — the window path's layout carries padding, junk grid
        positions and 4-bit digit fields and is not counted beyond this."""
        return self.a_bits * self.n * self.L.h * self.L.w * self.bs.packed_row_words(self.L.ic) * 4

    def tcw_item(self):
        L = self.L
        return dict(act_win=self.win, w_win=self.w_win, out=self.out, n=self.n, h=L.h, w=L.w, c=L.ic, oc=L.oc,
                    kh=L.k, kw=L.k, stride=L.s, pad=L.pad, w_enc=self.enc)

    def tcw_pack_item(self):
        L = self.L
        return dict(x=self.act, kh=L.k, kw=L.k, stride=L.s, pad=L.pad)

    def group_item(self):
        L = self.L
        return dict(act_packed=self.packed, w_tc=self.w_tc, out=self.out, n=self.n, h=L.h, w=L.w, c=L.ic, oc=L.oc,
                    kh=L.k, kw=L.k, stride=L.s, pad=L.pad, w_enc=self.enc)

    def host_buffers(self):
        return (self.act_cpu.contiguous().pin_memory(), torch.empty(self.out.shape, dtype=torch.int32).pin_memory(),
                torch.empty_like(self.act), torch.empty_like(self.out))

    def host_step(self, bufs):
        L = self.L
        ah, oh_, ad, od = bufs
        if self.path == "tc":
            self.bs.bitserial_conv2d_nhwc_tc_host(ah, self.a_bits, self.w_tc, self.w_bits, L.oc, L.k, L.k, L.s,
                                                  L.pad, oh_, ad, od, self.ws, tc_format=self.fmt)
        else:
            self.bs.bitserial_conv2d_nhwc_host(ah, self.a_bits, self.wp, self.w_bits, self.enc, L.oc, L.k, L.k, L.s,
                                               L.pad, oh_, ad, od, self.ws)


class ConvWorkload:
    """configs[0] (conv1), configs[2] (resnet1), configs[3] (resnet256)."""

    def __init__(self, args, rank, world, dev, layers, batch, config_id, name):
        self.args, self.dev, self.batch = args, dev, batch
        # batch-1 configs do not shard: N independent replicas ("replicas only")
        self.replicas = world if batch < world else 1
        lo, hi = (0, batch) if self.replicas > 1 else bsdist.shard_range(batch, rank, world)
        self.images = (lo, hi)
        enc = "bipolar" if args.bipolar else "unipolar"
        self.runs, self.layers = [], layers
        for li in layers:
            L = inputs.TABLE1[li]
            act, wt = inputs.conv_operands(L, batch, args.a_bits, args.w_bits,
                                           inputs.seed_for(config_id, args.a_bits, args.w_bits, enc, li))
            lpath = args.path
            if args.path == "hybrid":  # window path for the layers it runs faster, expansion kernel for the rest
                lpath = "tcw" if li in hybrid_tcw_layers(args) else "tc"
            self.runs.append(ConvLayerRun(L, act[lo:hi].contiguous(), wt, args.a_bits, args.w_bits, args.bipolar,
                                          dev, lpath, tc_fmt(args)))
        self.total_binops = self.replicas * sum(binops_conv(inputs.TABLE1[li], batch, args.a_bits, args.w_bits)
                                                for li in layers)
        self.config_id = config_id
        self.name = name
        self.graph_ok = True
        # pack/conv overlap across layers (two streams) for the tensor-core path
        self.overlap = args.path == "tc" and not args.no_overlap
        if self.overlap:
            self.side_stream = torch.cuda.Stream(device=dev)
            self.pack_events = [torch.cuda.Event() for _ in self.runs]
            self.pack_ctas = args.pack_ctas_per_sm * torch.cuda.get_device_properties(dev).multi_processor_count
            self.split_ctas = max(1, args.split_pack_ctas_per_sm) * torch.cuda.get_device_properties(dev).multi_processor_count
            self.conv_streams = args.conv_streams
            self.extra_conv_streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
            self.packs_first = args.packs_first
            # grouped convs: the layers split into `conv_groups` contiguous groups, each one
            # bs_bitserial_conv2d_nhwc_tc_group launch (0: one launch per layer)
            ng = min(args.conv_groups, len(self.runs))
            self.groups = ([list(range(len(self.runs)))[g * len(self.runs) // ng:(g + 1) * len(self.runs) // ng]
                            for g in range(ng)] if ng > 0 else [])
            if args.group_layers:  # explicit partition, e.g. "2|4,5,6,7,8,9,10,11,12"
                self.groups = [[self.layers.index(int(x)) for x in part.split(",")]
                               for part in args.group_layers.split("|")]
                assert sorted(i for grp in self.groups for i in grp) == list(range(len(self.runs)))
            self.group_items = [[self.runs[i].group_item() for i in grp] for grp in self.groups]
        if args.path in ("tcd", "tcw", "hybrid"):  # few pack + conv launches for every layer
            # every layer's activations and outputs live in one flat device buffer each (views), so the
            # end-to-end step moves its inputs and results with one copy per direction
            na = sum(r.act.numel() for r in self.runs)
            no = sum(r.out.numel() for r in self.runs)
            self.flat_act = torch.empty(na + 16 * len(self.runs), dtype=torch.uint8, device=dev)
            self.flat_out = torch.empty(no + 4 * len(self.runs), dtype=torch.int32, device=dev)
            oa = oo = 0
            for r in self.runs:
                a = self.flat_act[oa:oa + r.act.numel()].view(r.act.shape)
                a.copy_(r.act)
                r.act = a
                r.out = self.flat_out[oo:oo + r.out.numel()].view(r.out.shape)
                oa += (r.act.numel() + 15) // 16 * 16  # 16-byte aligned views
                oo += (r.out.numel() + 3) // 4 * 4
            self.tcd_items = [r.tcd_item() for r in self.runs] if args.path == "tcd" else None
            self.w_runs = [r for r in self.runs if r.path == "tcw"]
            self.t_runs = [r for r in self.runs if r.path == "tc"]
            self.tcw_items = [r.tcw_item() for r in self.w_runs]
            self.tcw_pack = [r.tcw_pack_item() for r in self.w_runs]
            self.tc_items = [r.group_item() for r in self.t_runs]
            if args.path == "hybrid":
                self.hy_streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
        if args.path == "small":  # every layer in ONE launch of the small-problem path (packing fused)
            self.small_items = [dict(act=r.act, w_packed=r.wp, out=r.out, w_enc=r.enc, oc=r.L.oc, kh=r.L.k, kw=r.L.k,
                                     stride=r.L.s, pad=r.L.pad) for r in self.runs]
        self.config = {
            "workload": f"{name}_a{args.a_bits}w{args.w_bits}_{enc}", "global_batch": batch, "layers": list(layers),
            "window_path_layers": ([r.L.name for r in self.runs if r.path == "tcw"] if args.path == "hybrid" else
                                   None),
            "layout": "NHWC/OHWI",
            "parallelism": (f"{world} independent replicas (batch 1 does not shard)" if self.replicas > 1 else
                            f"batch-sharded dp{world} (no collective)"),
            "rank0_images": [lo, hi],
            "step": self.describe_step(args),
            "path": args.path,
            "hybrid_order": ([args.hybrid_order, args.hybrid_pack_ctas_per_sm] if args.path == "hybrid" else None),
            "tc_format": args.tc_format if args.path in ("tc", "hybrid") else None,
            "conv_groups": (args.conv_groups if self.overlap else 0),
            "pack_group": bool(self.overlap and args.pack_group),
            "pack_split": bool(self.overlap and args.pack_group and args.pack_split and self.groups),
        }

    def describe_step(self, args):
        if args.path == "hybrid":
            return (f"layers {[r.L.name for r in self.runs if r.path == 'tcw']} on the window path (ONE "
                    "bs_digitpack_win_group + ONE bs_bitserial_conv2d_nhwc_tcw_group launch, own stream) beside layers "
                    f"{[r.L.name for r in self.runs if r.path == 'tc']} on the expansion kernel (ONE bs_bitpack_group "
                    "launch on a side stream, then ONE bs_bitserial_conv2d_nhwc_tc_group call); " +
                    {0: "the two packs start together",
                     1: "the bit-plane pack starts when the window pack ends, beside the window conv",
                     2: "the window pack starts when the bit-plane pack ends, beside the expansion conv"}[
                         args.hybrid_order] + "; weights packed and prepared once, untimed")
        if args.path == "tcw":
            return ("every layer's activations packed into its conv's window layout (zero-padded stride phases, 32-byte "
                    "swizzled digit rows, DESIGN.md R26) by ONE bs_digitpack_win_group launch, then every layer's conv "
                    "in ONE bs_bitserial_conv2d_nhwc_tcw_group launch (bulk-copied windows, each filter tap a shifted "
                    "shared-memory view, tcgen05 kind::mxf4; weights packed + prepared once, untimed)")
        if args.path == "tcd":
            return ("every layer's activations digit-packed by ONE bs_digitpack_group launch, then every layer's conv "
                    "in ONE bs_bitserial_conv2d_nhwc_tcd_group launch (TMA-fed tcgen05 kind::mxf4 on digit-packed "
                    "operands; weights packed + digit-prepared once, untimed)")
        if args.path == "small":
            return ("every layer's conv from raw uint8 codes in ONE bs_bitserial_conv2d_nhwc_i8_group launch (activation "
                    "packing fused in shared memory, AND+POPC, K slices summed through cluster shared memory; weights "
                    "packed once, untimed)")
        if args.path != "tc":
            return ("per layer: bitpack(act) + AND/POPC bitserial conv2d via bs_bitserial_conv2d_nhwc_i8 (weights "
                    "prepacked, untimed)")
        if args.no_overlap:
            return ("per layer: bitpack(act) + tensor-core bitserial conv2d via bs_bitserial_conv2d_nhwc_tc_i8 "
                    "(weights packed + plane-expanded once, untimed)")
        packs = ("the activations packed by one bs_bitpack_group launch per conv group, in group order [side stream]"
                 if args.pack_group and args.pack_split and self.groups else
                 "every layer's activations packed by ONE bs_bitpack_group launch [side stream]" if args.pack_group
                 else "per layer bs_bitpack [side stream]")
        convs = (f"the layers' tensor-core convs in {len(self.groups)} bs_bitserial_conv2d_nhwc_tc_group calls "
                 f"{[[self.layers[i] for i in g] for g in self.groups]} on alternating streams (each waits for its "
                 "members' packs)" if self.groups else
                 "per layer bs_bitserial_conv2d_nhwc_tc_prepared on alternating streams (each waits for its pack)")
        return f"{packs}; {convs} (weights packed + plane-expanded once, untimed)"

    def step(self):
        if self.args.path == "hybrid":
            bs = self.runs[0].bs
            main = torch.cuda.current_stream()
            s_w, s_p = self.hy_streams
            s_w.wait_stream(main)
            s_p.wait_stream(main)
            ho = self.args.hybrid_order
            if ho:  # one path's pack beside the OTHER path's conv instead of beside its pack
                sm = torch.cuda.get_device_properties(self.dev).multi_processor_count
                cap = self.args.hybrid_pack_ctas_per_sm * sm
                wpack = lambda: bs.digitpack_win_group(self.tcw_pack, self.args.a_bits,  # noqa: E731
                                                       outs=[r.win for r in self.w_runs])
                tpack = lambda c: bs.bitpack_group([r.act for r in self.t_runs], self.args.a_bits,  # noqa: E731
                                                   outs=[r.packed for r in self.t_runs], max_ctas=c)
                wconv = lambda: bs.bitserial_conv2d_nhwc_tcw_group(self.tcw_items, self.args.a_bits,  # noqa: E731
                                                                   self.args.w_bits)
                tconv = lambda: bs.bitserial_conv2d_nhwc_tc_group(self.tc_items, self.args.a_bits,  # noqa: E731
                                                                  self.args.w_bits, tc_format=tc_fmt(self.args))
                if ho == 1:  # window pack; then [window conv || bit-plane pack]; then expansion conv
                    with torch.cuda.stream(s_w):
                        wpack()
                    s_p.wait_stream(s_w)
                    with torch.cuda.stream(s_w):
                        wconv()
                    with torch.cuda.stream(s_p):
                        tpack(cap)
                        tconv()
                else:  # bit-plane pack; then [expansion conv || window pack (no cap option)]; then window conv
                    with torch.cuda.stream(s_p):
                        tpack(0)
                    s_w.wait_stream(s_p)
                    with torch.cuda.stream(s_p):
                        tconv()
                    with torch.cuda.stream(s_w):
                        wpack()
                        wconv()
                main.wait_stream(s_p)
                main.wait_stream(s_w)
                return
            with torch.cuda.stream(s_w):
                bs.digitpack_win_group(self.tcw_pack, self.args.a_bits, outs=[r.win for r in self.w_runs])
                bs.bitserial_conv2d_nhwc_tcw_group(self.tcw_items, self.args.a_bits, self.args.w_bits)
            with torch.cuda.stream(s_p):
                bs.bitpack_group([r.act for r in self.t_runs], self.args.a_bits, outs=[r.packed for r in self.t_runs])
            main.wait_stream(s_p)
            bs.bitserial_conv2d_nhwc_tc_group(self.tc_items, self.args.a_bits, self.args.w_bits,
                                              tc_format=tc_fmt(self.args))
            main.wait_stream(s_w)
            return
        if self.args.path == "tcw":
            bs = self.runs[0].bs
            bs.digitpack_win_group(self.tcw_pack, self.args.a_bits, outs=[r.win for r in self.runs])
            bs.bitserial_conv2d_nhwc_tcw_group(self.tcw_items, self.args.a_bits, self.args.w_bits)
            return
        if self.args.path == "tcd":
            bs = self.runs[0].bs
            bs.digitpack_group([r.act for r in self.runs], self.args.a_bits, outs=[r.dig for r in self.runs])
            bs.bitserial_conv2d_nhwc_tcd_group(self.tcd_items, self.args.a_bits, self.args.w_bits)
            return
        if self.args.path == "small":
            self.runs[0].bs.bitserial_conv2d_nhwc_i8_group(self.small_items, self.args.a_bits, self.args.w_bits)
            return
        if self.overlap:
            return self.step_overlapped()
        for r in self.runs:
            r.step()

    def step_overlapped(self):
        """Same work, two streams: the activation packing of every layer (bs_bitpack)
        runs on a side stream, each layer's tensor-core conv (bs_..._tc_prepared) waits
        only for its own layer's pack — packing of later layers overlaps the convs of
        earlier ones (the layers' inputs are independent).  Captured into the step's CUDA
        graph as parallel branches."""
        main = torch.cuda.current_stream()
        side = self.side_stream
        side.wait_stream(main)
        with torch.cuda.stream(side):
            if self.args.pack_group and self.args.pack_split and self.groups:
                # one grouped pack per conv group, in group order: a group's convs start as soon as
                # its own layers are packed while the later groups' packs run beside them
                for gi, grp in enumerate(self.groups):
                    # later groups' packs run beside the earlier groups' persistent convs: a capped
                    # grid of 128-thread CTAs fits next to a conv CTA on each SM
                    self.runs[0].bs.bitpack_group([self.runs[i].act for i in grp], self.args.a_bits,
                                                  outs=[self.runs[i].packed for i in grp],
                                                  max_ctas=0 if gi == 0 else self.split_ctas)
                    for i in grp:
                        self.pack_events[i].record(side)
            elif self.args.pack_group:  # every layer's activations packed by one launch
                self.runs[0].bs.bitpack_group([r.act for r in self.runs], self.args.a_bits,
                                              outs=[r.packed for r in self.runs])
                for e in self.pack_events:
                    e.record(side)
            for i, (r, e) in enumerate(zip(self.runs, self.pack_events)):
                if self.args.pack_group:
                    break
                # the first layer's pack has nothing to overlap: full grid; later packs run beside
                # the previous layer's persistent conv CTAs: a capped grid leaves them room
                r.pack_only(0 if i == 0 else self.pack_ctas)
                e.record(side)
        # the ten layers are independent problems (BASELINE configs[3]): convs alternate
        # between two streams so one layer's persistent CTAs start on the SMs the previous
        # layer's tail leaves idle (two conv CTAs never share an SM: smem + all of TMEM)
        conv_streams = [main] + self.extra_conv_streams[:self.conv_streams - 1]
        if self.packs_first:  # experiment: every pack before any conv
            for e in self.pack_events:
                main.wait_event(e)
        for s in conv_streams[1:]:
            s.wait_stream(main)
        if self.groups:  # one grouped tensor-core launch per group of layers
            for gi, (grp, items) in enumerate(zip(self.groups, self.group_items)):
                cs = conv_streams[gi % len(conv_streams)]
                for i in grp:
                    cs.wait_event(self.pack_events[i])
                with torch.cuda.stream(cs):
                    self.runs[0].bs.bitserial_conv2d_nhwc_tc_group(items, self.args.a_bits, self.args.w_bits,
                                                                   tc_format=tc_fmt(self.args))
        for i, (r, e) in enumerate(zip(self.runs, self.pack_events)):
            if self.groups:
                break
            cs = conv_streams[i % len(conv_streams)]
            cs.wait_event(e)
            with torch.cuda.stream(cs):
                r.conv_only()
        for s in conv_streams[1:]:
            main.wait_stream(s)
        main.wait_stream(side)

    def roofline_small(self, reps):
        """The small path's one launch per step (packing fused), timed as a whole."""
        ms = graph_launch_ms(self.step, reps)
        ops = sum(r.binops() for r in self.runs)
        nbytes = sum(r.act.numel() + r.wp.numel() * 4 + r.out.numel() * 4 for r in self.runs)
        return {"kind": "popc", "kernel": f"small_conv_kernel (one launch: {len(self.runs)} layers, fused packing, "
                                          "AND+POPC, cluster split-K)", "ops": ops, "ms": ms, "launches": 1,
                "bytes": nbytes, "breakdown": {"step_kernel_us": 1e3 * ms}}

    def roofline_tcd(self, reps):
        """The digit path's conv launch (all layers, one launch) and its pack launch, each
        graph-replayed; algorithmic bytes: activation digits + weight digits + int32 outputs."""
        bs = self.runs[0].bs
        bs.digitpack_group([r.act for r in self.runs], self.args.a_bits, outs=[r.dig for r in self.runs])
        conv = lambda: bs.bitserial_conv2d_nhwc_tcd_group(self.tcd_items, self.args.a_bits, self.args.w_bits)  # noqa
        pack = lambda: bs.digitpack_group([r.act for r in self.runs], self.args.a_bits,  # noqa
                                          outs=[r.dig for r in self.runs])
        ms, pms = graph_launch_ms(conv, reps), graph_launch_ms(pack, reps)
        nbytes = sum(r.dig.numel() + r.w_dig.numel() + r.out.numel() * 4 for r in self.runs)
        ops = sum(r.binops() for r in self.runs)
        return {"kind": "tensor", "kernel": f"tcd_conv_kernel (TMA-fed tcgen05 kind::mxf4 on digit-packed operands; "
                                            f"one launch for the {len(self.runs)} layers, rank 0)",
                "ops": ops, "ms": ms, "launches": 1, "bytes": nbytes,
                "breakdown": {"conv_group_us": 1e3 * ms, "digit_pack_group_us": 1e3 * pms}}

    def roofline_tcw(self, reps):
        """The window path's conv launch (all layers, one launch) and its pack launch, each
        graph-replayed; algorithmic bytes: bit-packed activations + packed weights + int32 outputs."""
        bs = self.runs[0].bs
        pack = lambda: bs.digitpack_win_group(self.tcw_pack, self.args.a_bits, outs=[r.win for r in self.runs])  # noqa
        conv = lambda: bs.bitserial_conv2d_nhwc_tcw_group(self.tcw_items, self.args.a_bits, self.args.w_bits)  # noqa
        pack()
        ms, pms = graph_launch_ms(conv, reps), graph_launch_ms(pack, reps)
        nbytes = sum(r.packed_bytes() + r.wp.numel() * 4 + r.out.numel() * 4 for r in self.runs)
        ops = sum(r.binops() for r in self.runs)
        return {"kind": "tensor", "kernel": f"tcw_conv_kernel (window path: bulk-copied windows, shifted-view taps, "
                                            f"tcgen05 kind::mxf4; one launch for the {len(self.runs)} layers, rank 0)",
                "ops": ops, "ms": ms, "launches": 1, "bytes": nbytes,
                "breakdown": {"conv_group_us": 1e3 * ms, "window_pack_group_us": 1e3 * pms}}

    def roofline_hybrid(self, reps):
        """The hybrid step's two conv calls (the window-path launch and the grouped expansion-kernel
        call) and two pack launches, each graph-replayed; algorithmic bytes per conv call: the
        bit-packed activations (window-path layers: the same bit-plane count, not the larger window
        layout), the weights (packed bit planes for the window path, the prepared form for the
        expansion kernel) and the int32 outputs."""
        bs, fmt = self.runs[0].bs, tc_fmt(self.args)
        wpack = lambda: bs.digitpack_win_group(self.tcw_pack, self.args.a_bits, outs=[r.win for r in self.w_runs])  # noqa
        tpack = lambda: bs.bitpack_group([r.act for r in self.t_runs], self.args.a_bits,  # noqa
                                         outs=[r.packed for r in self.t_runs])
        wconv = lambda: bs.bitserial_conv2d_nhwc_tcw_group(self.tcw_items, self.args.a_bits, self.args.w_bits)  # noqa
        tconv = lambda: bs.bitserial_conv2d_nhwc_tc_group(self.tc_items, self.args.a_bits, self.args.w_bits,  # noqa
                                                          tc_format=fmt)
        wpack()
        tpack()
        torch.cuda.synchronize()
        wms, tms = graph_launch_ms(wconv, reps), graph_launch_ms(tconv, reps)
        wpms, tpms = graph_launch_ms(wpack, reps), graph_launch_ms(tpack, reps)
        wbytes = sum(r.packed_bytes() + r.wp.numel() * 4 + r.out.numel() * 4 for r in self.w_runs)
        tbytes = sum(r.packed.numel() * 4 + r.w_tc.numel() + r.out.numel() * 4 for r in self.t_runs)
        per = [{"layers": [r.L.name for r in self.w_runs], "binops": sum(r.binops() for r in self.w_runs),
                "bytes": wbytes, "ms": wms},
               {"layers": [r.L.name for r in self.t_runs], "binops": sum(r.binops() for r in self.t_runs),
                "bytes": tbytes, "ms": tms}]
        return {"kind": "tensor", "kernel": "the step's conv launches: tcw_conv_kernel (window path, layers "
                                            f"{per[0]['layers']}) + tc_conv_kernel (expansion kernel, layers "
                                            f"{per[1]['layers']}), tcgen05 kind::mxf4, rank 0",
                "ops": per[0]["binops"] + per[1]["binops"], "ms": wms + tms, "launches": 2, "bytes": wbytes + tbytes,
                "per_layer": per,
                "breakdown": {"tcw_conv_us": 1e3 * wms, "tc_conv_group_us": 1e3 * tms, "window_pack_us": 1e3 * wpms,
                              "bitplane_pack_us": 1e3 * tpms}}

    def roofline(self, reps):
        """Per-launch device time of the pack and conv kernels of every layer: each
        kernel captured `reps` times back to back in a CUDA graph, timed with events on
        the stream that replays it (no host launch gaps), per launch = graph time / reps."""
        if self.args.path == "small":
            return self.roofline_small(reps)
        if self.args.path == "tcd":
            return self.roofline_tcd(reps)
        if self.args.path == "tcw":
            return self.roofline_tcw(reps)
        if self.args.path == "hybrid":
            return self.roofline_hybrid(reps)
        for r in self.runs:
            r.pack_only()
            r.conv_only()
        torch.cuda.synchronize()
        pack_ms = [graph_launch_ms(r.pack_only, reps) for r in self.runs]
        conv_ms = [graph_launch_ms(r.conv_only, reps) for r in self.runs]
        ops = sum(r.binops() for r in self.runs)
        pack_bytes = sum(r.act.numel() * (1 + r.a_bits / 8) for r in self.runs)
        tc = self.args.path == "tc"
        kname = (f"tc_conv_kernel (tcgen05 kind::{'mxf4' if self.args.tc_format == 'f4' else 'i8'};" if tc else
                 "popc_conv_kernel (")
        # algorithmic HBM bytes per conv launch: packed activations read once, weights
        # (prepared form) read once, int32 outputs written once
        conv_bytes = [r.packed.numel() * 4 + (r.w_tc.numel() if r.w_tc is not None else r.wp.numel() * 4)
                      + r.out.numel() * 4 for r in self.runs]
        res = {"kind": "tensor" if tc else "alu",
               "kernel": f"{kname} sum over the {len(self.runs)} layer launches of one step, rank 0)",
               "ops": ops, "ms": sum(conv_ms), "launches": len(self.runs), "bytes": sum(conv_bytes),
               "per_layer": [{"layer": li, "binops": r.binops(), "bytes": b, "ms": t}
                             for li, r, b, t in zip(self.layers, self.runs, conv_bytes, conv_ms)],
               "breakdown": {"layers": list(self.layers), "conv_us": [1e3 * t for t in conv_ms],
                             "pack_us": [1e3 * t for t in pack_ms],
                             "conv_binary_tops": [r.binops() / (t / 1e3) / 1e12 for r, t in zip(self.runs, conv_ms)],
                             "pack_gbs": pack_bytes / (sum(pack_ms) / 1e3) / 1e9,
                             "out_gbs": sum(r.out.numel() * 4 for r in self.runs) / (sum(conv_ms) / 1e3) / 1e9}}
        if tc and self.overlap and self.groups:
            # the step's launch configuration: one bs_bitserial_conv2d_nhwc_tc_group call per
            # group (a BN = 64 launch for OC <= 64 members, one persistent BN = 128 launch for
            # the rest), each timed as a whole (its members run concurrently inside it)
            bs, fmt = self.runs[0].bs, tc_fmt(self.args)
            fns = [lambda items=items: bs.bitserial_conv2d_nhwc_tc_group(items, self.args.a_bits, self.args.w_bits,
                                                                          tc_format=fmt) for items in self.group_items]
            n0 = bs.kernel_launches()
            for f in fns:
                f()
            launches = bs.kernel_launches() - n0
            torch.cuda.synchronize()
            gms = [graph_launch_ms(f, reps) for f in fns]
            per = [{"layers": [self.layers[i] for i in grp], "binops": sum(self.runs[i].binops() for i in grp),
                    "bytes": sum(conv_bytes[i] for i in grp), "ms": t} for grp, t in zip(self.groups, gms)]
            res.update(kernel=f"{kname} the step's {len(fns)} grouped calls ({launches} launches), rank 0)",
                       ms=sum(gms), launches=launches, per_layer=per)
            res["breakdown"]["group_us"] = [1e3 * t for t in gms]
            res["breakdown"]["groups"] = [[self.layers[i] for i in grp] for grp in self.groups]
        if tc and self.overlap and self.args.pack_group:
            pms = graph_launch_ms(lambda: self.runs[0].bs.bitpack_group(
                [r.act for r in self.runs], self.args.a_bits, outs=[r.packed for r in self.runs]), reps)
            res["breakdown"]["pack_group_us"] = 1e3 * pms
            res["breakdown"]["pack_group_gbs"] = pack_bytes / (pms / 1e3) / 1e9
        return res

    def e2e(self, steps):
        bufs = [r.host_buffers() for r in self.runs]
        if self.overlap:  # tensor-core path: one pipelined host-buffer call for all layers
            layers = [dict(act_host=b[0], out_host=b[1], act_dev=b[2], packed_dev=r.packed, out_dev=b[3], w_tc=r.w_tc,
                           oc=r.L.oc, kh=r.L.k, kw=r.L.k, stride=r.L.s, pad=r.L.pad, w_enc=r.enc)
                      for r, b in zip(self.runs, bufs)]
            # smallest upload first: the download stream (745 MB, the PCIe-bound part) starts sooner
            layers.sort(key=lambda d: d["act_host"].numel())
            bs, fmt = self.runs[0].bs, tc_fmt(self.args)

            def step():
                bs.bitserial_conv2d_nhwc_tc_host_group(layers, self.args.a_bits, self.args.w_bits, tc_format=fmt)
        elif self.args.path == "hybrid" and self.args.e2e_mode == "unified":
            # every layer, smallest upload first, through one pipeline of three streams: upload ->
            # pack + conv (bs_bitpack + bs_bitserial_conv2d_nhwc_tc_prepared, or bs_digitpack_win +
            # bs_bitserial_conv2d_nhwc_tcw) -> download, each layer's download as soon as its conv is done
            host = [(r.act_cpu.contiguous().pin_memory(), torch.empty(r.out.shape, dtype=torch.int32).pin_memory())
                    for r in self.runs]
            bufs = host
            bs = self.runs[0].bs
            su, sc, sd = (torch.cuda.Stream(device=self.dev) for _ in range(3))
            order = sorted(range(len(self.runs)), key=lambda i: self.runs[i].act.numel())
            ev_up = [torch.cuda.Event() for _ in order]
            ev_c = [torch.cuda.Event() for _ in order]
            widx = {id(r): k for k, r in enumerate(self.w_runs)}

            def step():
                for j, i in enumerate(order):
                    r, (ah, oh_) = self.runs[i], host[i]
                    with torch.cuda.stream(su):
                        r.act.copy_(ah, non_blocking=True)
                        ev_up[j].record(su)
                    sc.wait_event(ev_up[j])
                    with torch.cuda.stream(sc):
                        if r.path == "tcw":
                            k = widx[id(r)]
                            bs.digitpack_win_group([self.tcw_pack[k]], self.args.a_bits, outs=[r.win])
                            bs.bitserial_conv2d_nhwc_tcw_group([self.tcw_items[k]], self.args.a_bits, self.args.w_bits)
                        else:
                            r.pack_only()
                            r.conv_only()
                        ev_c[j].record(sc)
                    sd.wait_event(ev_c[j])
                    with torch.cuda.stream(sd):
                        oh_.copy_(r.out, non_blocking=True)
                sd.synchronize()
        elif self.args.path == "hybrid":
            # the expansion-kernel layers through the pipelined host-buffer call (uploads, pack + conv,
            # downloads on three streams), the window-path layers beside it on three more streams
            # (upload -> window pack + conv -> download): both share the PCIe link full duplex
            t_bufs = [r.host_buffers() for r in self.t_runs]
            layers = [dict(act_host=b[0], out_host=b[1], act_dev=b[2], packed_dev=r.packed, out_dev=b[3], w_tc=r.w_tc,
                           oc=r.L.oc, kh=r.L.k, kw=r.L.k, stride=r.L.s, pad=r.L.pad, w_enc=r.enc)
                      for r, b in zip(self.t_runs, t_bufs)]
            layers.sort(key=lambda d: d["act_host"].numel())
            w_host = [(r.act_cpu.contiguous().pin_memory(), torch.empty(r.out.shape, dtype=torch.int32).pin_memory())
                      for r in self.w_runs]
            bufs = [(b[0], b[1]) for b in t_bufs] + w_host
            bs, fmt = self.runs[0].bs, tc_fmt(self.args)
            su, sc, sd = (torch.cuda.Stream(device=self.dev) for _ in range(3))
            # per layer, smallest upload first (as the host-group call orders its layers): each
            # layer's download starts as soon as its own conv is done
            order = sorted(range(len(self.w_runs)), key=lambda i: self.w_runs[i].act.numel())
            ev_up = [torch.cuda.Event() for _ in order]
            ev_c = [torch.cuda.Event() for _ in order]

            def step():
                for j, i in enumerate(order):
                    r, (ah, oh_) = self.w_runs[i], w_host[i]
                    with torch.cuda.stream(su):
                        r.act.copy_(ah, non_blocking=True)
                        ev_up[j].record(su)
                    sc.wait_event(ev_up[j])
                    with torch.cuda.stream(sc):
                        bs.digitpack_win_group([self.tcw_pack[i]], self.args.a_bits, outs=[r.win])
                        bs.bitserial_conv2d_nhwc_tcw_group([self.tcw_items[i]], self.args.a_bits, self.args.w_bits)
                        ev_c[j].record(sc)
                    sd.wait_event(ev_c[j])
                    with torch.cuda.stream(sd):
                        oh_.copy_(r.out, non_blocking=True)
                bs.bitserial_conv2d_nhwc_tc_host_group(layers, self.args.a_bits, self.args.w_bits, tc_format=fmt)
                sd.synchronize()
        elif self.args.path in ("tcd", "tcw"):  # one upload of every layer's codes, the step, one download
            host_in = self.flat_act.cpu().pin_memory()
            host_out = torch.empty(self.flat_out.shape, dtype=torch.int32).pin_memory()
            bufs = [(host_in, host_out)]

            def step():
                self.flat_act.copy_(host_in, non_blocking=True)
                self.step()
                host_out.copy_(self.flat_out, non_blocking=True)
                torch.cuda.current_stream().synchronize()
        else:
            def step():
                for r, b in zip(self.runs, bufs):
                    r.host_step(b)
        step()
        bsdist.barrier()
        torch.cuda.synchronize()
        stream = torch.cuda.current_stream()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        bsdist.barrier()
        ms = e0.elapsed_time(e1) / steps
        return ms, sum(b[0].numel() for b in bufs), sum(b[1].numel() * 4 for b in bufs)

    def parity_check(self, rank, world):
        """EVERY output of the TIMED step (what the graph replays left in HBM) against the
        oracle on the same inputs: all of this rank's images, every layer, in blocks of
        32 images (the OpenMP oracle runs ~5 ms per image of the ten layers)."""
        import numpy as np

        import oracle
        a = self.args
        checked = mism = 0
        for r in self.runs:
            L = r.L
            for b0 in range(0, r.n, 32):
                b1 = min(r.n, b0 + 32)
                got = r.out[b0:b1].cpu().numpy()
                ref = oracle.conv2d_nhwc(r.act_cpu[b0:b1].numpy(), a.a_bits, r.wt_cpu.numpy(), a.w_bits, a.bipolar,
                                         stride=(L.s, L.s), pad=(L.pad, L.pad))
                checked += ref.size
                mism += int(np.count_nonzero(got != ref))
        lo, hi = self.images
        return checked, mism, f"all outputs of images [{lo}, {hi}) of layers {list(self.layers)}"

    def oracle_sample(self, images):
        """The oracle on `images` images of every layer (same seeds as the GPU arm)."""
        import oracle
        a = self.args
        enc = "bipolar" if a.bipolar else "unipolar"
        ops, t = 0, 0.0
        for li in self.layers:
            L = inputs.TABLE1[li]
            g = inputs.gen(inputs.seed_for(self.config_id, a.a_bits, a.w_bits, enc, li))
            act = inputs.codes((images, L.h, L.w, L.ic), a.a_bits, g).numpy()
            wt = inputs.codes((L.oc, L.k, L.k, L.ic), a.w_bits, g).numpy()
            t0 = time.perf_counter()
            oracle.conv2d_nhwc(act, a.a_bits, wt, a.w_bits, a.bipolar, stride=(L.s, L.s), pad=(L.pad, L.pad))
            t += time.perf_counter() - t0
            ops += binops_conv(L, images, a.a_bits, a.w_bits)
        return ops, t, f"{images} image(s) of layers {list(self.layers)}"

    def oracle_units(self, budget_s):
        ops1, t1, _ = self.oracle_sample(1)
        return max(1, min(self.batch, int(budget_s / max(t1, 1e-3))))


# ----------------------------------------------------------------------------- dense
class DenseWorkload:
    """configs[1] (gemv: M=1, N=K=4096) and configs[4] (gemm: M=N=K=size,
    row-sharded, NCCL all-gather of the int32 result)."""

    def __init__(self, args, rank, world, dev, m, n, k, config_id, name, gather):
        import paper_1810_11066_b200 as bs
        self.bs, self.args, self.dev = bs, args, dev
        self.m, self.n, self.k, self.gather, self.world = m, n, k, gather, world
        self.a_bits, self.w_bits = args.a_bits, args.w_bits
        self.enc = bs.BIPOLAR if args.bipolar else bs.UNIPOLAR
        enc = "bipolar" if args.bipolar else "unipolar"
        a, w = inputs.dense_operands(m, n, k, args.a_bits, args.w_bits,
                                     inputs.seed_for(config_id, args.a_bits, args.w_bits, enc))
        if gather and m % world:
            raise SystemExit(f"gemm rows {m} not divisible by {world} ranks")
        lo, hi = bsdist.shard_range(m, rank, world) if gather else (0, m)
        self.rows = (lo, hi)
        self.a_cpu = a[lo:hi].contiguous()
        self.a = self.a_cpu.to(dev)
        self.wp = bs.bitpack(w.to(dev), args.w_bits)  # untimed
        del w
        self.tc = args.path == "tc" and (hi - lo) > 8  # GEMV (m <= 8) stays on the HBM-bound matvec kernel
        self.fmt = tc_fmt(args)
        # the digit path (digit-packed operands, TMA-fed tcgen05 kernel) unless the I8 format or
        # the fused all-gather epilogue (a variant of the expansion kernel) is asked for
        self.digit = self.tc and args.tc_format == "f4" and not args.fused_gather
        self.w_tc = (bs.dense_tc_prepare_weights(self.wp, args.w_bits, self.enc, n, k, tc_format=self.fmt)
                     if self.tc and not self.digit else None)
        self.w_dig = bs.dense_tcd_prepare_weights(self.wp, args.w_bits, self.enc, n, k) if self.digit else None
        self.a_dig = (torch.empty(((args.a_bits + 1) // 2, hi - lo, bs.digit_row_bytes(k)), dtype=torch.uint8,
                                  device=dev) if self.digit else None)
        self.out = torch.empty((hi - lo, n), dtype=torch.int32, device=dev)
        # one rank: its row block IS the whole C (no exchange step, no copy)
        self.full = (torch.empty((m, n), dtype=torch.int32, device=dev) if world > 1 else self.out) if gather else None
        self.ws = torch.empty(max(16, bs.dense_workspace_bytes(hi - lo, k, args.a_bits)), dtype=torch.uint8, device=dev)
        kwp = bs.packed_row_words(k)
        self.packed = self.ws[:args.a_bits * (hi - lo) * kwp * 4].view(torch.int32).view(args.a_bits, hi - lo, kwp)
        self.replicas = 1 if gather else world
        # fused all-gather epilogue: C lives in symmetric memory; each rank's
        # tensor-core kernel stores its row block into every rank's copy over NVLink
        self.fused = None
        if gather and self.tc and args.fused_gather:
            self.fused = bsdist.FusedGather(m, n, lo, hi, dev)
        self.total_binops = 2 * m * n * k * args.a_bits * args.w_bits * self.replicas
        self.config_id, self.name = config_id, name
        self.graph_ok = not (gather and world > 1)
        self.config = {
            "workload": f"{name}_m{m}_n{n}_k{k}_a{args.a_bits}w{args.w_bits}_{enc}", "m": m, "n": n, "k": k,
            "parallelism": (f"row-sharded tp{world} + all_gather_into_tensor(int32 C) over NCCL" if gather else
                            "single GPU (replicas only)"),
            "step": ("bs_digitpack (activation digit packing) + bs_bitserial_dense_tcd (TMA-fed tensor-core dense)"
                     if self.digit else
                     "bs_bitserial_dense_tc_i8 (activation pack + tensor-core dense)" if self.tc else
                     "bs_bitserial_dense_i8 (activation pack + dense" + (", fused single launch" if (hi - lo) <= 8
                                                                         else "") + ")")
                    + (" + NCCL all-gather of C" if gather else ""),
            "path": ("tc-digit" if self.digit else "tc") if self.tc else ("gemv" if (hi - lo) <= 8 else "popc"),
        }
        if self.fused is not None:
            self.config["parallelism"] = (f"row-sharded tp{world}; all-gather fused into the tensor-core epilogue "
                                          f"({self.fused.describe()})")
            self.config["step"] = ("bitpack(A shard) + bs_bitserial_dense_tc_prepared_gather (C row block stored to "
                                   "every rank's symmetric-memory C) + device barrier")

    def step(self):
        if self.fused is not None:
            rows = self.rows[1] - self.rows[0]
            self.bs.bitpack(self.a, self.a_bits, out=self.packed)
            self.bs.bitserial_dense_tc_gather(self.packed, self.a_bits, self.w_tc, self.w_bits, rows, self.n, self.k,
                                              self.fused.local_block(), self.fused.peer_blocks(), tc_format=self.fmt,
                                              w_enc=self.enc)
            self.fused.barrier()
            return
        if self.digit:
            rows = self.rows[1] - self.rows[0]
            self.bs.digitpack(self.a, self.a_bits, out=self.a_dig)
            self.bs.bitserial_dense_tcd(self.a_dig, self.a_bits, self.w_dig, self.w_bits, rows, self.n, self.k,
                                        out=self.out, w_enc=self.enc)
        elif self.tc:
            self.bs.bitserial_dense_tc_i8(self.a, self.a_bits, self.w_tc, self.w_bits, self.n, out=self.out,
                                          workspace=self.ws, tc_format=self.fmt)
        else:
            self.bs.bitserial_dense_i8(self.a, self.a_bits, self.wp, self.w_bits, self.enc, self.n, out=self.out,
                                       workspace=self.ws)
        if self.gather and self.world > 1:
            bsdist.gather_rows(self.full, self.out)

    def roofline(self, reps):
        stream = torch.cuda.current_stream()
        rows = self.rows[1] - self.rows[0]
        gemv = rows <= 8

        def kernel():
            if gemv:
                self.bs.bitserial_dense_i8(self.a, self.a_bits, self.wp, self.w_bits, self.enc, self.n, out=self.out,
                                           workspace=self.ws)
            elif self.digit:
                self.bs.bitserial_dense_tcd(self.a_dig, self.a_bits, self.w_dig, self.w_bits, rows, self.n, self.k,
                                            out=self.out, w_enc=self.enc)
            elif self.tc:
                self.bs.bitserial_dense_tc_prepared(self.packed, self.a_bits, self.w_tc, self.w_bits, rows, self.n,
                                                    self.k, out=self.out, tc_format=self.fmt)
            else:
                self.bs.bitserial_dense(self.packed, self.a_bits, self.wp, self.w_bits, self.enc, rows, self.n,
                                        self.k, out=self.out, algo=self.bs.ALGO_POPC)
        if self.digit:
            self.bs.digitpack(self.a, self.a_bits, out=self.a_dig)
        elif not gemv:
            self.bs.bitpack(self.a, self.a_bits, out=self.packed)
        kernel()
        torch.cuda.synchronize()
        flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=self.dev)
        ms = 0.0
        for _ in range(reps):
            flush.zero_()
            e0, e1 = ev(), ev()
            e0.record(stream)
            kernel()
            e1.record(stream)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1) / reps
        comm_ms = None
        if self.gather and self.world > 1:
            e0, e1 = ev(), ev()
            bsdist.barrier()
            e0.record(stream)
            for _ in range(reps):
                bsdist.gather_rows(self.full, self.out)
            e1.record(stream)
            torch.cuda.synchronize()
            comm_ms = e0.elapsed_time(e1) / reps
        ops = 2 * rows * self.n * self.k * self.a_bits * self.w_bits
        if gemv:
            nbytes = self.wp.numel() * 4 + self.a.numel() + self.out.numel() * 4
            return {"kind": "hbm", "kernel": "gemv_kernel (fused pack + GEMV, one launch, cold L2)", "bytes": nbytes,
                    "ops": ops, "ms": ms, "breakdown": {"gemv_ms": ms}}
        if self.digit:
            return {"kind": "tensor", "ops": ops, "ms": ms, "launches": 1,
                    "kernel": "tcd_conv_kernel (TMA-fed tcgen05 kind::mxf4 on digit-packed operands, 128x224 tiles; "
                              "rank 0 shard)",
                    "bytes": self.a_dig.numel() + self.w_dig.numel() + self.out.numel() * 4,
                    "breakdown": {"dense_ms": ms, "allgather_ms": comm_ms}}
        return {"kind": "tensor" if self.tc else "alu",
                "kernel": (f"tc_conv_kernel (tcgen05 kind::{'mxf4' if self.args.tc_format == 'f4' else 'i8'}; dense = "
                           "1x1 implicit GEMM, rank 0 shard)" if self.tc else
                           "popc_conv_kernel (dense = 1x1 implicit GEMM, rank 0 shard)"), "ops": ops,
                "ms": ms, "launches": 1,
                "bytes": self.packed.numel() * 4 + (self.w_tc.numel() if self.tc else self.wp.numel() * 4)
                + self.out.numel() * 4,
                "breakdown": {"dense_ms": ms, "allgather_ms": comm_ms}}

    def e2e(self, steps):
        a_host = self.a_cpu.pin_memory()
        c_host = torch.empty((self.m if self.gather else self.out.shape[0], self.n), dtype=torch.int32).pin_memory()
        stream = torch.cuda.current_stream()

        def step():
            self.a.copy_(a_host, non_blocking=True)
            self.step()
            c_host.copy_(self.full if self.gather else self.out, non_blocking=True)
        step()
        torch.cuda.synchronize()
        bsdist.barrier()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        bsdist.barrier()
        return e0.elapsed_time(e1) / steps, a_host.numel(), c_host.numel() * 4

    def parity_check(self, rank, world):
        """Rows of the timed step's C against the oracle: every row of the GEMV; for the
        GEMM 64 rows spread over C plus the first row of EVERY rank's block (and the last
        row) of this rank's gathered C, so the exchange step is checked too."""
        import numpy as np

        import oracle
        enc = "bipolar" if self.args.bipolar else "unipolar"
        a, w = inputs.dense_operands(self.m, self.n, self.k, self.a_bits, self.w_bits,
                                     inputs.seed_for(self.config_id, self.a_bits, self.w_bits, enc))
        if self.gather:
            pick = sorted({bsdist.shard_range(self.m, r, self.world)[0] for r in range(self.world)} |
                          set(range(0, self.m, max(1, self.m // 64))) | {self.m - 1})
            full = self.fused.full if self.fused is not None else self.full
            got = full[pick].cpu().numpy()
        else:
            pick = list(range(self.m)) if self.m <= 8 else sorted(set(range(0, self.m, max(1, self.m // 64))) |
                                                                   {self.m - 1})
            got = self.out[pick].cpu().numpy()
        ref = oracle.dense(a[pick].numpy(), self.a_bits, w.numpy(), self.w_bits, self.args.bipolar)
        return ref.size, int(np.count_nonzero(got != ref)), f"rows {pick} of C"

    def oracle_sample(self, rows):
        import oracle
        a = self.args
        enc = "bipolar" if a.bipolar else "unipolar"
        am, w = inputs.dense_operands(self.m, self.n, self.k, a.a_bits, a.w_bits,
                                      inputs.seed_for(self.config_id, a.a_bits, a.w_bits, enc))
        am = am[:rows].numpy()
        w = w.numpy()
        t0 = time.perf_counter()
        oracle.dense(am, a.a_bits, w, a.w_bits, a.bipolar)
        t = time.perf_counter() - t0
        return 2 * rows * self.n * self.k * a.a_bits * a.w_bits, t, f"{rows} row(s) of the {self.m}x{self.n}x{self.k} " \
                                                                    "product"

    def oracle_units(self, budget_s):
        ops1, t1, _ = self.oracle_sample(1)
        return max(1, min(self.m, 256, int(budget_s / max(t1, 1e-4))))


def make_workload(args, rank, world, dev):
    if args.workload == "resnet256":
        return ConvWorkload(args, rank, world, dev, inputs.BASELINE_LAYERS, 256, 4, "resnet18_layers2-12_b256")
    if args.workload == "resnet1":
        return ConvWorkload(args, rank, world, dev, inputs.BASELINE_LAYERS, 1, 3, "resnet18_layers2-12_b1")
    if args.workload == "conv1":
        return ConvWorkload(args, rank, world, dev, (2,), 1, 1, "conv_l2_56x56x64_b1")
    if args.workload == "gemv":
        return DenseWorkload(args, rank, world, dev, 1, 4096, 4096, 2, "gemv", gather=False)
    if args.workload == "gemm":
        s = args.size
        return DenseWorkload(args, rank, world, dev, s, s, s, 5, "gemm", gather=True)
    raise SystemExit(f"unknown workload {args.workload}")


# ---------------------------------------------------------------------------- timing
def graph_launch_ms(fn, reps, trials=5):
    """Median per-launch ms of `fn` captured `reps` times in one CUDA graph."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        s.synchronize()
        ts = []
        for _ in range(trials):
            e0, e1 = ev(), ev()
            e0.record(s)
            g.replay()
            e1.record(s)
            s.synchronize()
            ts.append(e0.elapsed_time(e1) / reps)
    torch.cuda.current_stream().wait_stream(s)
    return sorted(ts)[len(ts) // 2]


def time_steps(step_fn, steps, warmup, dev, flush, use_graph):
    """W untimed warm-ups, then K steps each bracketed by CUDA events on the launching
    stream, the L2 flushed between steps outside the events; barrier + synchronize on
    both sides; returns the max-over-ranks mean ms/step."""
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
    evs = [(ev(), ev()) for _ in range(steps)]
    bsdist.barrier()
    torch.cuda.synchronize()
    for e0, e1 in evs:
        flush.zero_()
        e0.record(stream)
        run()
        e1.record(stream)
    torch.cuda.synchronize()
    bsdist.barrier()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / steps
    return bsdist.max_over_ranks(ms, dev), graph is not None


def run_ours(args):
    world, rank, local = bsdist.env()
    bsdist.init("nccl", local)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1810_11066_b200 as bs
    bs._load()
    peaks, peaks_src = measured_peaks()
    wl = make_workload(args, rank, world, dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    n0 = bs.kernel_launches()  # launches per step, counted by the library on one eager step
    wl.step()
    torch.cuda.synchronize()
    launches_per_step = bs.kernel_launches() - n0

    with ClockSampler(local) as clk:
        ms, graphed = time_steps(wl.step, args.steps, args.warmup, dev, flush,
                                 use_graph=wl.graph_ok and not args.no_graph)
    clocks = clk.summary()
    value = wl.total_binops / (ms / 1e3) / 1e12
    # the timing protocol's own floor: one tiny torch kernel timed exactly like a step (L2 flushed
    # before it, events around it) — what a batch-1 step cannot go below on this box
    tiny = torch.zeros(1, device=dev)
    floor_ms, _ = time_steps(lambda: tiny.add_(1), max(args.steps, 5), 3, dev, flush, use_graph=True)

    # self-check: the outputs the timed step left in HBM against the oracle (same inputs)
    parity = None
    if not args.no_parity:
        if world > 1 and "OMP_NUM_THREADS" not in os.environ:
            os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // world))
        n_chk, n_bad, what = wl.parity_check(rank, world)
        tot = torch.tensor([n_chk, n_bad], dtype=torch.int64, device=dev)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(tot)
        n_chk, n_bad = int(tot[0]), int(tot[1])
        parity = {"result": "bit-exact" if n_bad == 0 else f"MISMATCH n={n_bad}", "outputs_checked": n_chk,
                  "ranks": world, "rank0_checked": what + " of the timed step, vs the CPU oracle (int32, zero tolerance)"}

    roof = wl.roofline(10)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_max = clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz") or MAX_MHZ_FALLBACK
    r_popc = 64.0 * POPC_PER_CLK_PER_SM * sms * f_max * 1e6 / 1e12
    r_int = 2.0 * r_popc
    if roof["kind"] == "tensor":
        # binary dot products on the tensor cores.  I8 (kind::i8): one binary MAC per MMA MAC
        # (bit planes), peak = 2 x the measured bf16 peak (tools/mma_bench.cu: kind::i8
        # sustains exactly 2x the kind::f16 MACs per clock).  FP4 (kind::mxf4, default):
        # peak = 4 x bf16 (B200_PROFILING.md nominal 9 vs 2.25 PFLOP/s) and one MMA MAC
        # multiplies two radix-4 digits, i.e. A*W / (ceil(A/2)*ceil(W/2)) binary MACs, so the
        # tensor roofline is stated in MMA ops (= binary ops x digits/planes).  Burst figure.
        f4 = args.tc_format != "i8"
        ratio = 4.0 if f4 else 2.0
        peak = ratio * peaks["bf16_tflops"]
        hbm = peaks["hbm_gbs"]
        mma_per_bin = (((args.a_bits + 1) // 2) * ((args.w_bits + 1) // 2) / (args.a_bits * args.w_bits)) if f4 else 1.0
        achieved = roof["ops"] * mma_per_bin / (roof["ms"] / 1e3) / 1e12
        sustained = ratio * peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        # time model: each launch is bound by max(tensor time, HBM time of its algorithmic
        # bytes) — the int32 outputs (4 bytes per output) make the 1x1 and early layers
        # HBM-bound; the primary "bound" is the one that dominates summed over the launches
        t_tensor = roof["ops"] * mma_per_bin / (peak * 1e12) * 1e3
        t_hbm = roof["bytes"] / (hbm * 1e9) * 1e3
        per = roof.get("per_layer", [])
        t_roof = sum(max(x["binops"] * mma_per_bin / (peak * 1e12), x["bytes"] / (hbm * 1e9)) * 1e3 for x in per) \
            if per else \
            max(t_tensor, t_hbm)
        model = {"t_tensor_ms": t_tensor, "t_hbm_ms": t_hbm, "t_roof_ms": t_roof, "t_actual_ms": roof["ms"],
                 "frac": t_roof / roof["ms"],
                 "per_layer": [{"layer": x.get("layer", x.get("layers")), "t_us": 1e3 * x["ms"],
                                "t_tensor_us": 1e6 * x["binops"] * mma_per_bin / (peak * 1e12),
                                "t_hbm_us": 1e6 * x["bytes"] / (hbm * 1e9)} for x in per]}
        common = {"kernel": roof["kernel"], "traffic": None,
                  "mma_kind": "kind::mxf4 (E2M1 radix-4 digits, UE8M0 digit scales, FP32 accum)" if f4 else
                              "kind::i8 (0/1 bytes, int32 accum)",
                  "tensor": {"achieved": achieved, "peak": peak, "unit": "TFLOP/s", "unit_note": "MMA ops (2 x FP4 or I8 MACs)", "frac": achieved / peak,
                             "binary_tops": roof["ops"] / (roof["ms"] / 1e3) / 1e12,
                             "mma_ops_per_binary_op": mma_per_bin,
                             "peak_basis": f"{'FP4' if f4 else 'INT8'} dense tensor peak = {ratio:.0f} x bf16_tflops "
                                           f"({peaks['bf16_tflops']:.1f}, {peaks_src}); "
                                           + ("1 MMA MAC = 1 radix-4 digit pair = A*W/(ceil(A/2)*ceil(W/2)) binary MACs"
                                              if f4 else "1 binary MAC = 1 MMA MAC"),
                             "peak_sustained": sustained, "frac_sustained": achieved / sustained,
                             "frac_of_int8_peak": achieved / (2.0 * peaks["bf16_tflops"]),
                             "peak_nominal": 9000.0 if f4 else 4500.0,
                             "frac_of_nominal": achieved / (9000.0 if f4 else 4500.0),
                             "peak_clock": (2 if f4 else 1) * 8189.0 * 2 * sms * f_max * 1e6 / 1e12,
                             "frac_of_clock": achieved / ((2 if f4 else 1) * 8189.0 * 2 * sms * f_max * 1e6 / 1e12)},
                  "hbm": {"achieved": roof["bytes"] / (roof["ms"] / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                          "frac": roof["bytes"] / (roof["ms"] / 1e3) / 1e9 / hbm,
                          "algorithmic_bytes": roof["bytes"]},
                  "time_model": model, "r_popc": r_popc,
                  # binary ops over the integer-pipe (POPC) roofline, both in binary TOPS
                  "x_r_popc": roof["ops"] / (roof["ms"] / 1e3) / 1e12 / r_popc}
        if t_hbm >= t_tensor:  # HBM dominates summed over the step's launches
            roofline = dict(common, bound="hbm", achieved=common["hbm"]["achieved"], peak=hbm, unit="GB/s",
                            frac=common["hbm"]["frac"], peak_basis=f"HBM copy bandwidth, {peaks_src}")
        else:
            roofline = dict(common, bound="tensor", achieved=achieved, peak=peak, unit="TFLOP/s",
                            frac=achieved / peak, peak_basis=common["tensor"]["peak_basis"])
    elif roof["kind"] == "popc":  # one POPC per word pair (bipolar via the identity): the POPC-pipe roofline
        achieved = roof["ops"] / (roof["ms"] / 1e3) / 1e12
        roofline = {"bound": "alu", "achieved": achieved, "peak": r_popc, "unit": "binary TOPS",
                    "frac": achieved / r_popc, "traffic": None, "r_popc": r_popc, "kernel": roof["kernel"],
                    "peak_basis": f"POPC pipe (measured 16 /clk/SM, profiles/r01_int_pipe_rates.json): 64 binary ops "
                                  f"per POPC x 16 x {sms} SMs x {f_max:.0f} MHz",
                    "bytes": roof["bytes"], "hbm_frac": roof["bytes"] / (roof["ms"] / 1e3) / 1e9 / peaks["hbm_gbs"]}
    elif roof["kind"] == "alu":
        achieved = roof["ops"] / (roof["ms"] / 1e3) / 1e12
        roofline = {"bound": "alu", "achieved": achieved, "peak": r_int, "unit": "binary TOPS",
                    "frac": achieved / r_int, "traffic": None, "r_popc": r_popc, "frac_r_popc": achieved / r_popc,
                    "kernel": roof["kernel"],
                    "peak_basis": f"integer pipes (measured rates, profiles/r01_int_pipe_rates.json): per 32-bit word "
                                  f"pair 1 LOP3 + {{1 POPC | 2 LOP3}} balanced -> 32 word pairs/clk/SM x 64 binary "
                                  f"ops x {sms} SMs x {f_max:.0f} MHz (= 2 x R_popc)"}
    else:
        achieved = roof["bytes"] / (roof["ms"] / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / peaks["hbm_gbs"], "traffic": None, "kernel": roof["kernel"],
                    "peak_basis": f"HBM copy bandwidth, {peaks_src}",
                    "binary_tops": roof["ops"] / (roof["ms"] / 1e3) / 1e12}
    # the ncu traffic capture committed for this workload and path (the expansion-kernel step: no suffix)
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}{'' if args.path == 'tc' else '_' + args.path}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            roofline["traffic"] = json.load(f).get("dram_bytes_per_launch_unit")

    e2e = None
    if not args.no_e2e:
        ems, h2d, d2h = wl.e2e(max(1, min(args.steps, 5)))
        ems = bsdist.max_over_ranks(ems, dev)
        e2e = {"value": wl.total_binops / (ems / 1e3) / 1e12, "unit": "binary TOPS",
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * (1 if isinstance(wl, DenseWorkload)
                                                                               and wl.gather else world),
               "ms_per_step": ems}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        units = wl.oracle_units(10.0)
        ops, t, sample = wl.oracle_sample(units)
        cpu = {"value": ops / t / 1e12, "unit": "binary TOPS", "cores": oracle.num_threads(), "kind": "oracle",
               "sample": sample + " (bounded sample of the same workload, same seeds), OpenMP C oracle",
               "seconds": t, "cpu_model": cpu_model()}

    if rank == 0:
        cfg = dict(wl.config)
        cfg.update({"l2": f"{L2_FLUSH_BYTES >> 20} MiB buffer zeroed between timed steps (outside the events)",
                    "cuda_graph": graphed})
        line = {
            "metric": METRIC, "value": value, "unit": "binary TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "vs_baseline": None,
            "dtype": dtype_of(args, wl),
            "scaling": "weak" if getattr(wl, "replicas", 1) > 1 else "strong",
            "data": "synthetic (seeded uniform codes, PAPER.md Table 1 / BASELINE shapes; no dataset)",
            "config": cfg, "roofline": roofline,
            "breakdown": dict(roof.get("breakdown", {}), hbm_peak_gbs=peaks["hbm_gbs"], peaks_source=peaks_src),
            "clocks": clocks, "gpu_launches": launches_per_step * args.steps, "launches_per_step": launches_per_step,
            "timing_floor_us": {"value": 1e3 * floor_ms,
                                "what": "one 1-element torch kernel timed like a step (256 MiB L2 flush before it, "
                                        "CUDA events around it, CUDA graph): the protocol's fixed cost, included in "
                                        "ms_per_step"},
            "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def hybrid_tcw_layers(args):
    return [int(x) for x in args.tcw_layers.split(",") if x]


def dtype_of(args, wl):
    """The arithmetic the timed path computes in (not a precision claim)."""
    if args.path == "hybrid":
        return ("u8 codes -> window-layout e2m1 digit fields (window-path layers) | packed u32 bit-planes -> radix-4 "
                "e2m1 digits (expansion-kernel layers), x ue8m0 4^d scales on tcgen05 kind::mxf4 (fp32 accum, exact) "
                "-> i32")
    if args.path == "tcw":
        return ("u8 codes -> window-layout e2m1 digit fields (two bit-planes per nibble, 0.5 x {0..3}) x ue8m0 4^d "
                "scales on tcgen05 kind::mxf4 (fp32 accum, exact) -> i32")
    if getattr(wl, "digit", False) or args.path == "tcd":
        return ("u8 codes -> digit-packed e2m1 fields (two bit-planes per nibble, 0.5 x {0..3}) x ue8m0 4^d scales on "
                "tcgen05 kind::mxf4 (fp32 accum, exact) -> i32")
    if args.path == "tc":
        return ("u8 codes -> packed u32 bit-planes -> radix-4 e2m1 digits (two planes per nibble, 0.5 x {0..3}) x "
                "ue8m0 4^d scales on tcgen05 kind::mxf4 (fp32 accum, exact) -> i32" if args.tc_format == "f4" else
                "u8 codes -> packed u32 bit-planes -> i8 0/1 planes on tcgen05 kind::i8 -> i32")
    if args.path == "small":
        return "u8 codes -> u32 bit-planes packed in shared memory (AND/POPC) -> i32"
    return "u8 codes -> packed u32 bit-planes (AND/POPC) -> i32"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    """The reference arm of this tier: the CPU oracle, as it stands, on the host
    cores, each step a bounded sample of the same workload (rank 0 only)."""
    world, rank, _ = bsdist.env()
    if world > 1:  # under torchrun: a gloo group only to keep the ranks' exits together
        bsdist.init("gloo")
    if rank != 0:
        bsdist.barrier()
        return 0  # rank 0 alone runs the CPU oracle and prints
    import oracle
    oracle.build()
    wl = make_workload_cpu(args)
    units = max(1, wl.oracle_units(max(1.0, 60.0 / max(1, args.steps + args.warmup))))
    for _ in range(args.warmup):
        wl.oracle_sample(units)
    ts, ops, sample = [], 0, ""
    for _ in range(args.steps):
        ops, t, sample = wl.oracle_sample(units)
        ts.append(t)
    ms = 1e3 * sum(ts) / len(ts)
    value = ops / (ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "binary TOPS", "n_gpus": max(world, args.gpus), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u8 codes -> i32 (plain integer loops)", "data": "synthetic (seeded uniform codes)",
        "impl": "reference", "config": dict(wl.config, sample_per_step=sample),
        "cpu_baseline": {"value": value, "unit": "binary TOPS", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": sample + " per step (bounded sample of the workload; OpenMP C oracle)",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "binary TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    bsdist.barrier()
    return 0


def make_workload_cpu(args):
    """Workload descriptions for the oracle arm (no device allocations)."""
    class Conv(ConvWorkload):
        def __init__(self, layers, batch, cid, name):  # noqa: D401 — light init, oracle only
            self.args, self.layers, self.batch, self.config_id, self.name = args, layers, batch, cid, name
            enc = "bipolar" if args.bipolar else "unipolar"
            self.config = {"workload": f"{name}_a{args.a_bits}w{args.w_bits}_{enc}", "global_batch": batch,
                           "layers": list(layers)}

    class Dense(DenseWorkload):
        def __init__(self, m, n, k, cid, name):  # noqa: D401
            self.args, self.m, self.n, self.k, self.config_id, self.name = args, m, n, k, cid, name
            enc = "bipolar" if args.bipolar else "unipolar"
            self.config = {"workload": f"{name}_m{m}_n{n}_k{k}_a{args.a_bits}w{args.w_bits}_{enc}"}

    if args.workload == "resnet256":
        return Conv(inputs.BASELINE_LAYERS, 256, 4, "resnet18_layers2-12_b256")
    if args.workload == "resnet1":
        return Conv(inputs.BASELINE_LAYERS, 1, 3, "resnet18_layers2-12_b1")
    if args.workload == "conv1":
        return Conv((2,), 1, 1, "conv_l2_56x56x64_b1")
    if args.workload == "gemv":
        return Dense(1, 4096, 4096, 2, "gemv")
    return Dense(args.size, args.size, args.size, 5, "gemm")


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(n, argv=None):
    """`bench.py --gpus N` without torchrun: re-run this script as N ranks on one node
    (torch.distributed.run, rendezvous on 127.0.0.1), exactly as the driver launches it;
    rank 0 prints the JSON line.  Returns torchrun's exit status."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + \
        list(sys.argv[1:] if argv is None else argv)
    return subprocess.call(cmd)


def build_parser():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="resnet256", choices=["resnet256", "resnet1", "conv1", "gemv", "gemm"])
    ap.add_argument("--size", type=int, default=8192, help="gemm: M = N = K")
    ap.add_argument("--a-bits", type=int, default=2)
    ap.add_argument("--w-bits", type=int, default=1)
    ap.add_argument("--unipolar", dest="bipolar", action="store_false")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-overlap", action="store_true", help="pack and conv of every layer in one stream")
    ap.add_argument("--packs-first", action="store_true", help="overlapped step variant: all packs before any conv")
    ap.add_argument("--conv-streams", type=int, default=2, choices=[1, 2, 3],
                    help="overlapped step: convs of consecutive (independent) layers on 1 or 2 streams")
    ap.add_argument("--no-pack-group", dest="pack_group", action="store_false",
                    help="tensor-core path: one bs_bitpack launch per layer instead of one bs_bitpack_group launch")
    ap.add_argument("--pack-split", action="store_true",
                    help="one pack launch per conv group (later ones capped to fit beside the running convs) instead "
                         "of one for every layer (measured slower: profiles/r02e_step_sweep.jsonl)")
    ap.add_argument("--split-pack-ctas-per-sm", type=int, default=1,
                    help="split packs after the first: grid cap in 128-thread CTAs per SM")
    ap.add_argument("--group-layers", default="",
                    help="explicit conv groups as layer lists, e.g. '2|4,5,6,7,8,9,10,11,12' (overrides --conv-groups)")
    ap.add_argument("--conv-groups", type=int, default=2,
                    help="tensor-core path: layers per step in this many grouped launches (0: one launch per layer)")
    ap.add_argument("--pack-ctas-per-sm", type=int, default=0,
                    help="overlapped packs: grid cap in CTAs per SM (0 = library choice)")
    ap.add_argument("--tc-format", choices=["f4", "i8"], default="f4",
                    help="tensor-core operand format: block-scaled FP4 (default) or INT8")
    ap.add_argument("--e2e-mode", choices=["split", "unified"], default="unified",
                    help="--path hybrid e2e: split = the host-group call for the expansion-kernel layers beside a "
                         "window-path pipeline; unified = one per-layer pipeline for all layers")
    ap.add_argument("--tcw-layers", default="2,5,6,8",
                    help="--path hybrid: the layers on the window path (measured best partition, profiles/r02w_hybrid*)")
    ap.add_argument("--hybrid-order", type=int, default=1, choices=[0, 1, 2],
                    help="--path hybrid step composition: 1 (default) = window pack, then the bit-plane pack beside the "
                         "window conv (its 320-thread CTAs leave room on every SM), then the expansion conv; 0 = the two "
                         "packs side by side, then the two convs; 2 = window pack beside the expansion conv "
                         "(profiles/r02zj_hybrid_order.jsonl: 0.2357 / 0.2425 / 0.263 ms)")
    ap.add_argument("--hybrid-pack-ctas-per-sm", type=int, default=0,
                    help="--hybrid-order 1: grid cap of the bit-plane pack in CTAs per SM (0 = library choice)")
    ap.add_argument("--path", choices=["auto", "tc", "tcd", "tcw", "hybrid", "popc", "small"], default="auto",
                    help="conv/GEMM kernel: tensor-core bitserial (tc), the digit path (tcd), the window path (tcw), the "
                         "AND/POPC integer-pipe kernel, the one-launch small-problem path, or hybrid (--tcw-layers on "
                         "the window path, the rest on tc); auto = small for conv1, tcw for resnet1, hybrid for "
                         "resnet256, else tc")
    ap.add_argument("--fused-gather", action="store_true",
                    help="gemm, N>1: all-gather fused into the tensor-core epilogue over symmetric memory (SURVEY 8 f2)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle check of the timed step's outputs")
    return ap


def resolve_path(args):
    if args.path == "auto":  # measured: small ties the window path on the single batch-1 layer, the window path wins
        # the ten-layer batch-1 step (two launches; 20.4 vs 22.5 us for the digit path), the hybrid (layers 2, 5, 6, 8
        # on the window path beside the expansion kernel) the batch-256 step (0.242 vs 0.270 ms; profiles/r02v8_*)
        args.path = {"conv1": "small", "resnet1": "tcw", "resnet256": "hybrid"}.get(args.workload, "tc")
    return args


def main():
    args = resolve_path(build_parser().parse_args())
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:  # not launched by torchrun: launch N ranks (one per GPU) ourselves
        return relaunch(args.gpus)
    if world and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with --nproc-per-node {args.gpus}")
    if args.impl == "ours" and args.warmup < 3:
        args.warmup = 3
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
