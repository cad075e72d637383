"""`python -m paper_2008_11326_b200 gpp-run`: the reference's caller contract
(rooflab/cli.py:126-186; test_cli.py:78-119): usage errors exit 2 before any
GPU work (CPU), results and metrics with exit 0, divergence exit 1 (GPU)."""

import json

import pytest

from paper_2008_11326_b200 import cli


def test_usage_errors_exit_2(capsys):
    for argv in (["gpp-run", "--versions", "v99", "--dims", "4", "4", "64"],
                 ["gpp-run", "--dims", "0", "4", "64"],
                 ["gpp-run", "--dims", "4", "4", "64", "--trace"],
                 ["gpp-run", "--dims", "4", "4", "64", "--simulate", "desk"]):
        with pytest.raises(SystemExit) as info:
            cli.main(argv)
        assert info.value.code == 2
    capsys.readouterr()


@pytest.mark.gpu
def test_gpp_run_writes_metrics(tmp_path, capsys):
    code = cli.main(["gpp-run", "--dims", "8", "8", "64", "--seed", "1", "--versions", "v0,v5,v8",
                     "--out", str(tmp_path)])
    out = capsys.readouterr().out
    assert code == 0
    assert "all 3 versions within rtol 1e-10 of reference" in out
    records = json.loads((tmp_path / "metrics.json").read_text())
    assert [r["label"] for r in records] == ["v0", "v5", "v8"]
    assert records[0]["system"] == "synthetic-8x8x64-seed1"
    assert all(r["runtime"] > 0 for r in records)


@pytest.mark.gpu
def test_gpp_run_rtol_failure_path(capsys):
    code = cli.main(["gpp-run", "--dims", "4", "4", "64", "--seed", "1", "--versions", "v0,v8",
                     "--rtol", "0"])
    assert code == 1
    assert "diverge" in capsys.readouterr().err
