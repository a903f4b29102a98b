"""GPU: cclp::run_race over the B200 run_pdhg (librace_gpu.so) against the
same race over the reference's CPU run_pdhg (librace_cpu.so). north_star:
the final crossover basis must be identical as an index set and the
objective must agree to 1e-9."""
import pytest

from integration import race
from paper_2510_24429_b200 import lpgen

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (race.available("gpu") and race.available("cpu")),
                                 reason="oracle/_ref race libraries not built")]


@pytest.mark.parametrize("mode", ["baseline", "concurrent"])
def test_gpu_race_two_var(mode):
    out = race.run_race(lpgen.two_var_lp(), kind="gpu", mode=mode)
    assert out["status"] == "solved"
    assert out["objective"] == pytest.approx(2.0, abs=1e-6)


@pytest.mark.parametrize("seed", [3, 4])
def test_gpu_race_basis_matches_cpu_race(seed):
    lp = lpgen.transportation_lp(20, 30, seed=seed)
    g = race.run_race(lp, kind="gpu", mode="concurrent")
    c = race.run_race(lp, kind="cpu", mode="concurrent")
    assert g["status"] == c["status"] == "solved"
    assert g["basic"] == c["basic"]
    assert g["objective"] == pytest.approx(c["objective"], rel=1e-9, abs=1e-9)


def test_gpu_race_baseline_equals_concurrent_basis():
    lp = lpgen.transportation_lp(20, 30, seed=5)
    b = race.run_race(lp, kind="gpu", mode="baseline")
    c = race.run_race(lp, kind="gpu", mode="concurrent")
    assert b["winner"] == "main"
    assert b["basic"] == c["basic"]
    assert b["objective"] == pytest.approx(c["objective"], rel=1e-9)


def test_cli_solve_on_gpu(tmp_path):
    from integration import cli
    lp = lpgen.transportation_lp(20, 30, seed=3)
    cli.write_mps(lp, str(tmp_path / "t.mps"), "T")
    rc, g = cli.solve_file(str(tmp_path / "t.mps"), "concurrent", pdhg="gpu")
    rc2, c = cli.solve_file(str(tmp_path / "t.mps"), "concurrent", pdhg="cpu")
    assert rc == rc2 == 0
    assert g["objective"] == pytest.approx(c["objective"], rel=1e-9)


def test_cli_solve_cscb_on_gpu(tmp_path):
    """Binary CSC ingest through the CLI with the B200 PDHG: same objective as
    the MPS file of the same LP with the reference CPU PDHG."""
    from integration import cli
    from paper_2510_24429_b200.lp import write_cscb
    lp = lpgen.transportation_lp(20, 30, seed=4)
    cli.write_mps(lp, str(tmp_path / "t.mps"), "T")
    write_cscb(lp, str(tmp_path / "t.cscb"))
    rc, g = cli.solve_file(str(tmp_path / "t.cscb"), "concurrent", pdhg="gpu")
    rc2, c = cli.solve_file(str(tmp_path / "t.mps"), "concurrent", pdhg="cpu")
    assert rc == rc2 == 0
    assert g["objective"] == pytest.approx(c["objective"], rel=1e-9)
