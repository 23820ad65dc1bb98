"""One rank's shard of the multi-GPU bench step on one GPU (what `bench.py --gpus N` runs per rank):
build the workload for (rank, world), run the hybrid step, check every output of the shard against
the oracle.  Prints one JSON line per (rank, world)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for world, rank in ((2, 1), (4, 3), (8, 7)):
    args = bench.resolve_path(bench.build_parser().parse_args([]))
    dev = torch.device("cuda", 0)
    wl = bench.make_workload(args, rank, world, dev)
    wl.step()
    torch.cuda.synchronize()
    n, bad, what = wl.parity_check(rank, world)
    print(json.dumps({"world": world, "rank": rank, "path": args.path, "images": wl.images, "checked": n, "bad": bad}),
          flush=True)
