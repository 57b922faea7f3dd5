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


BENCH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bench")
BENCH_CASES = ("dual_fixed_bw", "dual_median_order", "dual_linear_nodiff")


def test_bench_config_schema():
    from paper_2501_07145_b200.cli import BENCH_SCHEMA
    cfg = validate_gram_config({"bench.methods": "dual_dp", "bench.n_list": [4, 8]}, "bench")
    assert cfg["bench.methods"] == ["dual_dp"] and cfg["bench.n_list"] == [4, 8]
    assert cfg["kernel.static.bandwidth"] == "median" and cfg["bench.wall_time"] is True
    assert set(cfg) == set(BENCH_SCHEMA) | {"command"}
    with pytest.raises(ConfigError, match="bench.methods: expected one of"):
        validate_gram_config({"bench.methods": "exact"}, "bench")
    with pytest.raises(ConfigError, match="bench.l_list: expected an integer >= 2"):
        validate_gram_config({"bench.l_list": 1}, "bench")


def test_bench_primal_methods_are_outside_the_path(tmp_path, capsys):
    cfg = tmp_path / "p.cfg"
    cfg.write_text("command = bench\nbench.methods = dual_dp, trp\n")
    assert main(["bench", "--config", str(cfg), "--output", str(tmp_path / "b.csv")]) == 1
    assert "outside the B200 dual path" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("name", BENCH_CASES)
def test_cli_bench_csv_bytes_match_reference(tmp_path, name):
    """`bench` with wall_time = false: every byte of the reference's CSV (record
    layout, F = N, flop_count and peak_bytes_est of the analytic model)."""
    out = tmp_path / "bench.csv"
    rc = main(["bench", "--config", os.path.join(BENCH, f"{name}.cfg"), "--output", str(out)])
    assert rc == 0
    assert out.read_bytes() == open(os.path.join(BENCH, f"{name}.out.csv"), "rb").read()


@pytest.mark.gpu
def test_run_bench_dual_dp_wall_time():
    from paper_2501_07145_b200.benchmarks import BenchSettings, run_bench
    from paper_2501_07145_b200.sequences import SeedStream
    recs = run_bench(BenchSettings(methods=("dual_dp", "dual_pde"), n_list=(16,), l_list=(32,),
                                   m_list=(3,), dim=4, bandwidth=1.0), SeedStream(5))
    assert [r.method for r in recs] == ["dual_dp", "dual_pde"]
    assert all(r.wall_ms > 0 and r.F == 16 and r.mape is None for r in recs)
