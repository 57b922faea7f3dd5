"""The `gram` CLI (cli.py:133-144) and its wire formats, against files the
reference CLI produced (tests/golden/make_cli_golden.py)."""

import os
import shutil

import numpy as np
import pytest

from paper_2501_07145_b200.cli import load_config, main, parse_config_text, validate_gram_config
from paper_2501_07145_b200.errors import ConfigError, ParseError
from paper_2501_07145_b200.wire import (load_sequences_csv, read_matrix_csv, tabulate,
                                        write_matrix_csv)

CLI = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
CASES = ("rbf_levelwise", "median_linear_global", "linear_none", "pde_global")


def test_tabulate_matches_reference():
    z = np.load(os.path.join(CLI, "tabulated.npz"))
    for name in CASES:
        b = tabulate(*load_sequences_csv(os.path.join(CLI, f"{name}.csv")))
        assert np.array_equal(b.data, z[f"{name}__data"]), name
        assert np.array_equal(b.ids, z[f"{name}__ids"]), name


def test_matrix_csv_bytes_match_reference(tmp_path):
    for name in CASES:
        ref = os.path.join(CLI, f"{name}.out.csv")
        out = tmp_path / f"{name}.csv"
        write_matrix_csv(out, read_matrix_csv(ref))
        assert out.read_bytes() == open(ref, "rb").read(), name


def test_config_parsing_and_validation():
    cfg = load_config(os.path.join(CLI, "median_linear_global.cfg"))
    assert cfg["kernel.static.bandwidth"] == "median" and cfg["kernel.order"] == 2
    assert cfg["kernel.difference"] is True and cfg["seed"] == 0
    assert parse_config_text("a = 1, 2.5, x\nb = none # c\n") == {"a": [1, 2.5, "x"], "b": None}
    with pytest.raises(ParseError, match="line 2: duplicate key 'a'"):
        parse_config_text("a = 1\na = 2")
    with pytest.raises(ParseError, match="line 1: expected 'key = value'"):
        parse_config_text("novalue")
    with pytest.raises(ConfigError, match="unknown config key 'kernel.bogus'"):
        validate_gram_config({"input": "x", "kernel.bogus": 1})
    with pytest.raises(ConfigError, match="kernel.n_levels: expected an integer >= 0"):
        validate_gram_config({"input": "x", "kernel.n_levels": -1})
    with pytest.raises(ConfigError, match="input: required"):
        validate_gram_config({})
    with pytest.raises(ConfigError, match="config file says 'synth'"):
        validate_gram_config({"command": "synth", "input": "x"})


def test_cli_error_exit_codes(tmp_path, capsys):
    bad = tmp_path / "bad.cfg"
    bad.write_text("command = gram\ninput = x.csv\nkernel.order = 0\n")
    assert main(["gram", "--config", str(bad)]) == 2
    assert "kernel.order: expected a positive integer or none" in capsys.readouterr().err
    other = tmp_path / "o.cfg"
    other.write_text("synth.n = 3\n")
    assert main(["synth", "--config", str(other)]) == 2
    missing = tmp_path / "m.cfg"
    missing.write_text(f"input = {tmp_path / 'nope.csv'}\n")
    assert main(["gram", "--config", str(missing)]) == 1  # OSError -> 1 (cli.py:267-269)
    broken = tmp_path / "b.csv"
    broken.write_text("seq_id,step,c0\n1,0,0.5\n1,x,1.0\n")
    cfgb = tmp_path / "c.cfg"
    cfgb.write_text(f"input = {broken}\n")
    assert main(["gram", "--config", str(cfgb)]) == 2
    assert "line 3: step must be an integer" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_cli_gram_matches_reference(tmp_path, name, precision):
    for ext in (".cfg", ".csv"):
        shutil.copy(os.path.join(CLI, name + ext), tmp_path / (name + ext))
    cwd = os.getcwd()
    os.chdir(tmp_path)
    try:
        rc = main(["gram", "--config", f"{name}.cfg", "--output", "K.csv",
                   "--precision", precision])
    finally:
        os.chdir(cwd)
    assert rc == 0
    K = read_matrix_csv(tmp_path / "K.csv")
    R = read_matrix_csv(os.path.join(CLI, f"{name}.out.csv"))
    # float64 kernels (fp64, and the pde path at either setting): the reference's 1e-10;
    # the FP32 fused path: the north star's 1e-4 (these cases include unnormalised ones)
    tol = 1e-10 if precision == "fp64" or name.startswith("pde") else 1e-4
    assert K.shape == R.shape
    assert np.allclose(K, R, rtol=tol, atol=tol * 1e-2), np.abs(K - R).max()
