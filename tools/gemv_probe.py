"""Latency probe of the batch-1 dense path (configs[1]: m=1, n=k=4096, A2W1 bipolar): the fused
GEMV launch timed warm (graph-replayed), cold (256 MiB L2 flush before each, events around the
launch, as bench.py does) and, for calibration, an empty-ish 1-block torch kernel under the same
cold protocol.  Prints one JSON object."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402
from bench import graph_launch_ms  # noqa: E402

dev = "cuda"
g = inputs.gen(5)
a = inputs.codes((1, 4096), 2, g).to(dev)
w = inputs.codes((4096, 4096), 1, g).to(dev)
wp = bs.bitpack(w, 1)
out = torch.empty((1, 4096), dtype=torch.int32, device=dev)
ws = torch.empty(max(16, bs.dense_workspace_bytes(1, 4096, 2)), dtype=torch.uint8, device=dev)
f = lambda: bs.bitserial_dense_i8(a, 2, wp, 1, bs.BIPOLAR, 4096, out=out, workspace=ws)  # noqa: E731
tiny = torch.zeros(1, device=dev)
t = lambda: tiny.add_(1)  # noqa: E731
res = {"warm_graph_us": 1e3 * graph_launch_ms(f, 50), "tiny_warm_graph_us": 1e3 * graph_launch_ms(t, 50)}
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for name, fn in (("gemv", f), ("tiny", t)):
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    res[f"{name}_cold_events_us_median"] = ts[len(ts) // 2]
print(json.dumps(res))
