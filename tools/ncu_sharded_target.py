"""Minimal driver for ncu: P row-block shards of a config on one GPU, a few
iterations (tools/probe_sharded.py measures the same path with events)."""
import os
import sys

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import PdhgConfig, ShardedEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
its = int(sys.argv[3]) if len(sys.argv) > 3 else 3
with ShardedEngine(lpgen.make_config(cfg), P) as se:
    se.begin(PdhgConfig())
    se.advance(its)
