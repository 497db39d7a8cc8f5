"""Reporting front end (reference src/bench.py, src/cli.py): records, renderers,
exit codes; GPU: a real solve and a 2-way parallel suite through the CLI."""
import json

import pytest

from paper_2307_16830_b200 import cli
from paper_2307_16830_b200.grids import tiled_case
from paper_2307_16830_b200.report import BenchRecord, render_csv, render_text


def test_record_roundtrip_and_renderers():
    r = BenchRecord(case="c", n_var=3, n_con=2, iterations=5, status="optimal", objective=1.5,
                    violation=1e-9, seconds={"total": 0.1, "ad": 0.01, "linear": 0.05, "internal": 0.04})
    assert BenchRecord.from_json(r.to_json()) == r
    csv_text = render_csv([r])
    assert csv_text.splitlines()[0].startswith("case,n_var,n_con")
    assert "optimal" in render_text([r, BenchRecord(case="bad", status="failed")])


def test_cli_usage_and_input_errors(tmp_path, capsys):
    assert cli.main(["solve", str(tmp_path / "missing.m")]) == 1
    assert cli.main(["solve", "x.m", "--tol", "-1"]) == 1
    assert cli.main(["bogus"]) == 1
    bad = tmp_path / "bad.m"
    bad.write_text("function mpc = bad\nmpc.baseMVA = 100;\n")
    assert cli.main(["solve", str(bad)]) == 1


@pytest.mark.gpu
def test_cli_solve_and_parallel_suite(tmp_path, capsys):
    a, b = tmp_path / "t1.m", tmp_path / "t2.m"
    a.write_text(tiled_case(1))
    b.write_text(tiled_case(2))
    assert cli.main(["solve", str(a), "--format", "json", "--tol", "1e-6"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["status"] == "optimal" and rec["iterations"] > 0
    man = tmp_path / "cases.txt"
    man.write_text("t1.m\n# comment\nt2.m\n")
    assert cli.main(["suite", str(man), "--parallel", "2", "--out", str(tmp_path / "o")]) == 0
    recs = json.loads((tmp_path / "o" / "records.json").read_text())
    assert [r["status"] for r in recs] == ["optimal", "optimal"]
