"""CPU: the bench/solve CLI (SPEC "[MODULE] bench_cli"):
shifted geometric mean and win/loss examples, summary invariants, report
round trips, and `solve` / `bench` end to end with the reference's CPU PDHG
(the GPU variant is the same code with --pdhg gpu)."""
import json
import math
import os

import pytest

from integration import cli, race
from paper_2510_24429_b200 import lpgen


def test_shifted_geomean_examples():
    assert cli.shifted_geomean([3.7]) == pytest.approx(3.7)
    assert cli.shifted_geomean([1, 4], 1.0) == pytest.approx(math.sqrt(10) - 1)
    assert cli.shifted_geomean([0, 0], 1.0) == pytest.approx(0.0)
    assert cli.shifted_geomean([1, 5, 2]) == pytest.approx(cli.shifted_geomean([5, 2, 1]))
    with pytest.raises(ValueError):
        cli.shifted_geomean([])


def test_classify_examples():
    assert cli.classify_win_loss(10, 8.9) == "win"
    assert cli.classify_win_loss(10, 9.5) == "tie"
    assert cli.classify_win_loss(10, 11.1) == "loss"


def test_summary_invariants_and_reports():
    recs = []
    for i, (b, c, w) in enumerate([(10, 5, "1e-02"), (4, 4, "main"), (2, 3, "1e-03")]):
        recs.append(dict(model=f"m{i}", mode="baseline", wall_s=b, status="solved", winner="main"))
        recs.append(dict(model=f"m{i}", mode="concurrent", wall_s=c, status="solved", winner=w))
    s = cli.summarize(recs)
    assert s["wins"] + s["losses"] + s["ties"] == s["models"] == 3
    assert (s["wins"], s["losses"], s["ties"]) == (1, 1, 1)
    assert sum(s["histogram"].values()) == 3 and list(s["histogram"])[-1] == "main"
    assert s["performance_ratio"] == pytest.approx(s["sgm"]["baseline"] / s["sgm"]["concurrent"])
    assert json.loads(cli.emit_report(s, "json"))["models"] == 3
    assert len(cli.emit_report(s, "csv").strip().splitlines()) == len(recs) + 1
    same = cli.summarize([dict(r, wall_s=1.0) for r in recs])
    assert same["performance_ratio"] == pytest.approx(1.0) and same["ties"] == 3
    with pytest.raises(ValueError):
        cli.emit_report(s, "xml")


@pytest.mark.skipif(not race.available("cpu"), reason="oracle/_ref race libraries not built")
def test_solve_and_bench_end_to_end(tmp_path):
    for seed in (3, 4):
        cli.write_mps(lpgen.transportation_lp(8, 12, seed=seed), str(tmp_path / f"t{seed}.mps"),
                      f"T{seed}")
    basis, sol = tmp_path / "b.txt", tmp_path / "s.txt"
    rc = cli.main(["solve", str(tmp_path / "t3.mps"), "--pdhg", "cpu", "--json",
                   "--write-basis", str(basis), "--write-solution", str(sol)])
    assert rc == 0
    assert basis.read_text().startswith("* basis") and sol.read_text().startswith("* objective")
    assert cli.main(["solve", str(tmp_path / "missing.mps"), "--pdhg", "cpu"]) == 4
    (tmp_path / "bad.mps").write_text("ROWS\n Q R1\nENDATA\n")
    assert cli.main(["solve", str(tmp_path / "bad.mps"), "--pdhg", "cpu"]) == 4
    os.remove(tmp_path / "bad.mps")
    out = tmp_path / "r.json"
    assert cli.main(["bench", str(tmp_path), "--pdhg", "cpu", "--out", str(out),
                     "--csv", str(tmp_path / "r.csv")]) == 0
    rep = json.loads(out.read_text())
    assert rep["models"] == 2 and len(rep["records"]) == 4
    assert all(r["status"] == "solved" for r in rep["records"])


def test_solve_cscb_matches_mps(tmp_path, capsys):
    """`solve model.cscb` (binary CSC ingest) reaches the same optimum and
    basis as `solve model.mps` of the same LP."""
    from paper_2510_24429_b200.lp import write_cscb
    lp = lpgen.transportation_lp(8, 12, seed=5)
    cli.write_mps(lp, str(tmp_path / "t.mps"), "T")
    write_cscb(lp, str(tmp_path / "t.cscb"))
    outs = []
    for f in ("t.mps", "t.cscb"):
        assert cli.main(["solve", str(tmp_path / f), "--pdhg", "cpu", "--json"]) == 0
        outs.append(json.loads(capsys.readouterr().out.strip().splitlines()[-1]))
    a, b = outs
    assert a["status"] == b["status"] == "solved"
    assert (a["rows"], a["cols"]) == (b["rows"], b["cols"])
    assert math.isclose(a["objective"], b["objective"], rel_tol=1e-9, abs_tol=1e-9)
    (tmp_path / "bad.cscb").write_bytes(b"CCLPCSC1" + bytes(8))
    assert cli.main(["solve", str(tmp_path / "bad.cscb"), "--pdhg", "cpu"]) == 4
