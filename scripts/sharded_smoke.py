"""Run the sharded bench path (paper_1802_02619_b200.sharded.bench_main) under torchrun
on however many GPUs the box has (1 here): checks the JSON line end to end."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_02619_b200 import sharded  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--config", default="C5")
ap.add_argument("--scale", type=int, default=20_000_000)
ap.add_argument("--no-e2e", action="store_true")
sharded.bench_main(ap.parse_args())
