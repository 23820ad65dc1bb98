"""Per-layer timing of the window pack (bs_digitpack_win) at batch 256, A2: bytes read (the input
pixels the conv's phases keep) + bytes written (the layout), GB/s.  Prints one JSON object."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402
from bench import graph_launch_ms  # noqa: E402

res = []
for li in inputs.BASELINE_LAYERS:
    L = inputs.TABLE1[li]
    act = inputs.codes((256, L.h, L.w, L.ic), 2, inputs.gen(li)).cuda()
    out = bs.digitpack_win(act, 2, L.k, L.k, L.s, L.pad)
    ms = graph_launch_ms(lambda: bs.digitpack_win(act, 2, L.k, L.k, L.s, L.pad, out=out), 20)
    read = act.numel() // (4 if (L.k == 1 and L.s == 2) else 1)
    packed = bs.bitpack(act.view(-1, L.ic), 2)
    pms = graph_launch_ms(lambda: bs.bitpack(act.view(-1, L.ic), 2, out=packed), 20)
    res.append({"layer": li, "win_us": 1e3 * ms, "win_gbs": (read + out.numel()) / ms / 1e6,
                "bitpack_us": 1e3 * pms, "bitpack_gbs": (act.numel() + packed.numel() * 4) / pms / 1e6})
print(json.dumps(res, indent=1))
