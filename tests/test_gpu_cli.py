"""CLI on the GPU: bench, the compare-modes tripwire (pass and a perturbed
stream that must trip it), a config-file run of the fixed-source slab."""

import pytest

from paper_2403_12345_b200 import cli

pytestmark = pytest.mark.gpu


def test_bench_and_compare_modes(tmp_path):
    common = ["--gridpoints", "40", "--n-axial", "4", "--out", str(tmp_path), "--quiet"]
    assert cli.main(["bench", "--particles", "2000", "--inactive", "1", "--active", "2"] + common) == 0
    assert (tmp_path / "bench.csv").exists()
    assert cli.main(["compare-modes", "--particles", "500", "--caps", "64,500",
                     "--tally-modes", "fused"] + common) == 0
    assert cli.main(["compare-modes", "--particles", "500", "--caps", "64",
                     "--tally-modes", "fused", "--perturb-stream", "7"] + common) == cli.EXIT_TRIPWIRE


def test_run_config_fixed_source(tmp_path):
    cfg = tmp_path / "slab.cfg"
    cfg.write_text("preset = shielding_slab\ngridpoints = 100\nrun_mode = fixed_source\n"
                   "particles = 2000\ninactive = 0\nactive = 2\nmesh = 2,2,6\n")
    assert cli.main(["run", str(cfg), "--out", str(tmp_path), "--quiet"]) == 0
    assert "leaks" in (tmp_path / "summary.txt").read_text()
