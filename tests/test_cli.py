"""Front end (cli.py / config.py, mirroring eventmc's): parsing, problem
assembly, exit codes -- CPU only; the GPU runs are in test_gpu_cli.py."""

import os

import pytest

from paper_2403_12345_b200 import cli, config


def test_config_parse_and_errors(tmp_path):
    v = config.parse_config_text("particles = 300\n# c\nsort = off\nmesh = 4,4,2\nrun_mode = fixed_source\n")
    assert v == {"particles": 300, "sort": False, "mesh": "4,4,2", "run_mode": "fixed_source"}
    with pytest.raises(config.ConfigurationError, match="line 1: unknown config key 'bogus'"):
        config.parse_config_text("bogus = 1")
    with pytest.raises(config.ConfigurationError, match="needs an integer"):
        config.parse_config_text("particles = many")
    p = config.build_problem({"preset": "shielding_slab", "gridpoints": 50, "run_mode": "fixed_source",
                              "mesh": "3,3,4"})
    assert p.pincell.is_slab and p.pincell.boundary == "vacuum" and p.run.mesh == (3, 3, 4)
    p = config.build_problem({"preset": "pwr_assembly", "gridpoints": 50})
    assert p.pincell.lattice == 17


def test_cli_exit_codes(tmp_path, capsys):
    bad = tmp_path / "bad.cfg"
    bad.write_text("particles = 10\nnonsense = 1\n")
    assert cli.main(["run", str(bad), "--out", str(tmp_path)]) == cli.EXIT_CONFIG
    assert "unknown config key" in capsys.readouterr().err
    out = tmp_path / "lib.bin"
    assert cli.main(["generate-library", "--nuclides", "4", "--gridpoints", "20", "--materials", "2",
                     "--per-material", "2", "-o", str(out), "--quiet"]) == cli.EXIT_OK
    assert os.path.getsize(out) > 0
