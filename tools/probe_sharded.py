"""Sharded-solve probe on one GPU: the single-device engine vs P shards in one
process (device-copy exchanges: halo or all-gather) vs the NCCL transport
with one rank. With P shards sharing one GPU the per-iteration time is the
sum of the P shards' kernels plus the exchanges, i.e. the compute-side cost
of sharding; `halo volume` is the per-iteration exchange in doubles (vs the
all-gather's (P-1) x (m + n))."""
import os
import sys

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import (Engine, PdhgConfig, ShardedEngine,  # noqa: E402
                                        nccl_unique_id)

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 100
shard_counts = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2, 4, 8]
halos = sys.argv[4].split(",") if len(sys.argv) > 4 else ["1", "0"]
with_nccl = len(sys.argv) <= 5 or sys.argv[5] != "no-nccl"
lp = lpgen.make_config(cfg)
B = 24 * lp.nnz + 20 * (lp.m + lp.n) + 8
eng = Engine(lp)
eng.begin(PdhgConfig())
eng.advance(20)
ms = eng.advance(its)
print(f"{cfg} single: {ms/its*1e3:.1f} us/it ({B/(ms/its*1e-3)/1e9:.0f} GB/s)", flush=True)
eng.close()
for halo in halos:
    os.environ["CCLP_CU_DEV_KNOBS"] = "1"
    os.environ["CCLP_CU_HALO"] = halo
    for P in shard_counts:
        with ShardedEngine(lp, P) as se:
            se.begin(PdhgConfig())
            se.advance(20)
            ms = se.advance(its)
            d = se.describe()
            print(f"{cfg} local shards P={P} halo={'on' if d['halo_x'] else 'off'}: {ms/its*1e3:.1f} us/it, "
                  f"x/y exchange {d['halo_x_volume']}/{d['halo_y_volume']} doubles "
                  f"(all-gather {(P-1)*(lp.n)}/{(P-1)*lp.m})", flush=True)
if not with_nccl:
    sys.exit(0)
with ShardedEngine(lp, 1, rank=0, nranks=1, nccl_id=nccl_unique_id()) as se:
    se.begin(PdhgConfig())
    se.advance(20)
    ms = se.advance(its)
    print(f"{cfg} NCCL transport, 1 rank: {ms/its*1e3:.1f} us/it", flush=True)
