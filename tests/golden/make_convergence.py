"""Convergence fixtures for BASELINE configs, generated from the REFERENCE ITSELF.

Run in the build container (needs oracle/_ref, i.e. /root/reference at build
time; CPU minutes per config):

    make -C oracle ref restate
    python tests/golden/make_convergence.py C1 1e-6      # ~3 min
    python tests/golden/make_convergence.py C2 1e-4      # ~5 min

For each (config, eps_rel) it runs
  * the reference's own run_pdhg (oracle/_ref/libcclp_ref.so: proj/src/pdhg.cpp
    compiled unmodified) -> stop, iterations, restarts, final report, seconds;
  * the plain-C restatement (oracle/liboracle.so) with its restart trace ->
    the list of restart iterations;
asserts that the two agree (same stop, iterations and restarts), and writes
tests/golden/convergence_<config>_<eps>.json. tests/test_gpu_convergence.py
checks the B200 engine against these numbers (iterations within 5 %,
north_star) on the GPU box, where /root/reference does not exist.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference, Restatement  # noqa: E402
from paper_2510_24429_b200 import lpgen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def fixture_path(config: str, eps: float) -> str:
    return os.path.join(HERE, f"convergence_{config}_{eps:.0e}.json")


def main(config: str, eps: float, which: str = "both") -> None:
    lp = lpgen.make_config(config)
    tol = dict(eps_rel=eps)
    out = dict(config=config, eps_rel=eps, m=lp.m, n=lp.n, nnz=int(lp.nnz),
               generator=f"paper_2510_24429_b200.lpgen.make_config('{config}')")
    if which in ("both", "ref"):
        t0 = time.time()
        ref = Reference().run_pdhg(lp, tol=tol, keep_snapshots=False)
        out["reference"] = dict(stop=ref["stop"], iterations=ref["iterations"],
                                restarts=ref["restarts"], report=ref["report"],
                                seconds=ref["seconds"], wall=time.time() - t0)
        print(config, eps, "reference", ref["stop"], ref["iterations"], ref["restarts"],
              f"{time.time() - t0:.1f}s", flush=True)
    if which in ("both", "restate"):
        t0 = time.time()
        rst = Restatement().run_pdhg(lp, tol=tol, restart_cap=4096)
        out["restatement"] = dict(stop=rst["stop"], iterations=rst["iterations"],
                                  restarts=rst["restarts"], report=rst["report"],
                                  restart_iters=[int(v) for v in rst["restart_iters"]],
                                  wall=time.time() - t0)
        print(config, eps, "restatement", rst["stop"], rst["iterations"], rst["restarts"],
              f"{time.time() - t0:.1f}s", flush=True)
    path = fixture_path(config, eps)
    if which != "both":  # partial run: merge into an existing fixture
        if os.path.exists(path):
            with open(path) as f:
                prev = json.load(f)
            prev.update(out)
            out = prev
    if "reference" in out and "restatement" in out:
        r, s = out["reference"], out["restatement"]
        assert (r["stop"], r["iterations"], r["restarts"]) == (s["stop"], s["iterations"], s["restarts"]), \
            (r, s)
        out["agree"] = True
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "both")
