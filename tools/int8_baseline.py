"""Paper-analog baselines on B200 (PAPER.md:717-729 compares
bitserial matmul against an 8-bit integer baseline): the same M = N = K products
computed by the int8 tensor cores (torch._int_mm -> cuBLASLt IMMA) and bf16
(torch.matmul), on the decoded integer values, next to our bitserial path.

Reported per (size, A, W): device ms (events, median, cold L2), int8/bf16 TOPS,
and "equivalent binary TOPS" = 2*M*N*K*A*W / t so the three are comparable with the
bench's metric; the int8 result is checked equal to the bitserial one on sampled rows.

    python tools/int8_baseline.py > gpurun_out/int8_baseline.json
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402


def timeit(fn, reps=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    res = []
    for size in (4096, 8192, 16384):
        for a_bits, w_bits in ((1, 1), (2, 1), (4, 2)):
            a, w = inputs.dense_operands(size, size, size, a_bits, w_bits, seed=size + 10 * a_bits + w_bits)
            a_d, w_d = a.cuda(), w.cuda()
            # bipolar weight values 2c - (2^W - 1), activations unsigned codes
            a8 = a_d.to(torch.int8)
            w8 = (2 * w_d.to(torch.int16) - ((1 << w_bits) - 1)).to(torch.int8)
            wp = bs.bitpack(w_d, w_bits)
            out = torch.empty((size, size), dtype=torch.int32, device="cuda")
            t_bs = timeit(lambda: bs.bitserial_dense_i8(a_d, a_bits, wp, w_bits, bs.BIPOLAR, size, out=out))
            w8t = w8.t()
            c8 = torch._int_mm(a8, w8t)
            t_i8 = timeit(lambda: torch._int_mm(a8, w8t))
            rows = [0, size // 3, size - 1]
            same = bool(torch.equal(c8[rows], out[rows]))
            ab, wb = a8.to(torch.bfloat16), w8.to(torch.bfloat16).t()
            t_bf = timeit(lambda: ab @ wb)
            mnk = size ** 3
            eq = 2 * mnk * a_bits * w_bits
            res.append({"size": size, "a_bits": a_bits, "w_bits": w_bits, "encoding": "bipolar",
                        "bitserial_ms": t_bs, "int8_ms": t_i8, "bf16_ms": t_bf,
                        "bitserial_binary_tops": eq / t_bs / 1e9, "int8_equiv_binary_tops": eq / t_i8 / 1e9,
                        "bf16_equiv_binary_tops": eq / t_bf / 1e9, "int8_tops": 2 * mnk / t_i8 / 1e9,
                        "bf16_tflops": 2 * mnk / t_bf / 1e9, "int8_equals_bitserial_on_sampled_rows": same,
                        "speedup_bitserial_over_int8": t_i8 / t_bs})
            del a8, w8, ab, wb, c8, out
            torch.cuda.empty_cache()
    print(json.dumps({"note": "int8 / bf16 = cuBLAS(Lt) via torch on decoded values (library baselines, not the "
                              "product path); bitserial = this repo's bs_bitserial_dense_i8 (pack + AND/POPC)",
                      "results": res}))


if __name__ == "__main__":
    main()
