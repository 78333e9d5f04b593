"""The full north_star C4 sweep (10k shapes) once, on the GPUs of this node
(same code path as bench.py's c4_sweep key, which defaults to a 2000-shape
sample to keep the default bench run within minutes):
  python scripts/c4_full.py [N_SHAPES]           # 1 GPU
  torchrun --nproc-per-node N scripts/c4_full.py  # sharded"""
import argparse
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
rank, world, local = bench.dist_init()
dev = torch.device("cuda", local)
P = bench.measured_peaks()["bf16_tflops"] * 1e12
out = bench.c4_sweep(argparse.Namespace(c4_shapes=n), rank, world, dev, P)
if rank == 0:
    print(json.dumps(out))
