"""`gram` and `bench` commands of the reference CLI on the B200 path
(cli.py:133-144, 197-214, config.py).

    python -m paper_2501_07145_b200 gram --config run.cfg [--seed S] [--output K.csv]
                                         [--threads N] [--precision fp32|fp64]
    python -m paper_2501_07145_b200 bench --config sweep.cfg [--output bench.csv] ...

Reads the reference's `key = value` config (config.py:47-76 parsing, the
`gram` schema of config.py:157-171, 213-226 with the same defaults, casts and
messages), loads and tabulates the sequence CSV named by `input`, evaluates
the Gram with `sig_kernel_gram` on the GPU and writes the headerless matrix
CSV. Exit codes as in cli.py:252-270: 2 for config/parse errors, 1 for other
library, value and OS errors. `--threads` is accepted for compatibility and
ignored (the device path has no host thread pool). `--precision` is this
build's extra flag (default fp32: the fused kernels; fp64: the float64 kernel).
`bench` runs the reference's sweep (config.py:217-232 schema) for its dual
cells (benchmarks.run_bench, `bench.methods` of dual_dp / dual_pde) and
writes the bench CSV. The reference's other commands (synth, features, mape,
classify) are outside this path and exit 2 with a message.
"""

from __future__ import annotations

import argparse
import sys

from .config import KERNEL_KINDS, KernelConfig, StaticKernelSpec
from .errors import ConfigError, ParseError, SigkernError
from .benchmarks import BENCH_METHODS, BenchSettings, run_bench, write_bench_csv
from .kernels import ALGORITHMS, sig_kernel_gram
from .sequences import SeedStream
from .static_kernels import median_heuristic
from .wire import load_sequences_csv, tabulate, write_matrix_csv

COMMANDS = ("synth", "gram", "features", "mape", "bench", "classify")  # config.py:26
NORMALIZATIONS = ("none", "levelwise", "global")


def _scalar(tok: str):
    t = tok.strip()
    low = t.lower()
    if low in ("true", "false"):
        return low == "true"
    if low in ("none", "null"):
        return None
    for cast in (int, float):
        try:
            return cast(t)
        except ValueError:
            pass
    return t


def parse_config_text(text: str) -> dict:
    """`key = value` lines, `#` comments, comma lists, typed scalars."""
    out = {}
    for n, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ParseError(f"expected 'key = value', got {line!r}", line=n)
        key, _, val = (s.strip() for s in line.partition("="))
        if not key:
            raise ParseError("missing key before '='", line=n)
        if not val:
            raise ParseError(f"missing value for key {key!r}", line=n)
        if key in out:
            raise ParseError(f"duplicate key {key!r}", line=n)
        if "," in val:
            items = [v.strip() for v in val.split(",")]
            if not all(items):
                raise ParseError(f"empty element in list value for {key!r}", line=n)
            out[key] = [_scalar(v) for v in items]
        else:
            out[key] = _scalar(val)
    return out


def _bad(key, v, want):
    raise ConfigError(f"{key}: expected {want}, got {v!r}")


def _choice(opts):
    def f(k, v):
        return v if isinstance(v, str) and v in opts else _bad(k, v, f"one of {', '.join(opts)}")
    return f


def _int(lo=None, hi=None):
    def f(k, v):
        if isinstance(v, bool) or not isinstance(v, int):
            _bad(k, v, "an integer")
        if lo is not None and v < lo:
            _bad(k, v, f"an integer >= {lo}")
        if hi is not None and v > hi:
            _bad(k, v, f"an integer <= {hi}")
        return v
    return f


def _num(positive=False):
    def f(k, v):
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            _bad(k, v, "a number")
        if positive and not v > 0:
            _bad(k, v, "a positive number")
        return float(v)
    return f


def _str(k, v):
    return v if isinstance(v, str) else _bad(k, v, "a string")


def _bool(k, v):
    return v if isinstance(v, bool) else _bad(k, v, "true or false")


def _order(k, v):
    if v is None:
        return None
    if isinstance(v, bool) or not isinstance(v, int) or v < 1:
        _bad(k, v, "a positive integer or none")
    return v


def _bandwidth(k, v):
    if isinstance(v, str):
        return v if v == "median" else _bad(k, v, 'a positive number or "median"')
    return _num(positive=True)(k, v)


GRAM_SCHEMA = {
    "seed": (_int(0, 2 ** 64 - 1), 0),
    "output": (_str, None),
    "input": (_str, None),
    "kernel.static.kind": (_choice(KERNEL_KINDS), "rbf"),
    "kernel.static.scale": (_num(positive=True), 1.0),
    "kernel.static.degree": (_int(1), 3),
    "kernel.static.gamma": (_num(), 1.0),
    "kernel.static.bandwidth": (_bandwidth, 1.0),
    "kernel.static.alpha": (_num(positive=True), 1.0),
    "kernel.n_levels": (_int(0), 5),
    "kernel.order": (_order, 1),
    "kernel.difference": (_bool, True),
    "kernel.normalization": (_choice(NORMALIZATIONS), "none"),
    "kernel.algorithm": (_choice(ALGORITHMS), "dp"),
}


def _list_of(cast):
    def f(k, v):
        return [cast(k, item) for item in (v if isinstance(v, list) else [v])]
    return f


BENCH_SCHEMA = {  # config.py:217-232
    "seed": (_int(0, 2 ** 64 - 1), 0),
    "output": (_str, None),
    "kernel.static.kind": (_choice(KERNEL_KINDS), "rbf"),
    "kernel.static.bandwidth": (_bandwidth, "median"),
    "bench.methods": (_list_of(_choice(BENCH_METHODS)), list(BENCH_METHODS)),
    "bench.n_list": (_list_of(_int(1)), [10]),
    "bench.l_list": (_list_of(_int(2)), [100]),
    "bench.dq_list": (_list_of(_int(1)), [100]),
    "bench.m_list": (_list_of(_int(0)), [5]),
    "bench.dim": (_int(1), 5),
    "bench.order": (_order, 1),
    "bench.difference": (_bool, True),
    "bench.mape": (_bool, False),
    "bench.n_seeds": (_int(1), 1),
    "bench.wall_time": (_bool, True),
}

SCHEMAS = {"gram": GRAM_SCHEMA, "bench": BENCH_SCHEMA}
_REQUIRED = {"gram": ("input",)}


def validate_gram_config(raw: dict, command: str = "gram") -> dict:
    """config.py:230-267 for the `gram` and `bench` commands."""
    file_cmd = raw.get("command")
    if file_cmd is not None and not isinstance(file_cmd, str):
        raise ConfigError(f"command: expected one of {', '.join(COMMANDS)}, got {file_cmd!r}")
    cmd = command if command is not None else file_cmd
    if cmd is None:
        raise ConfigError("command: missing (set the 'command' key or pass it on the CLI)")
    if cmd not in COMMANDS:
        raise ConfigError(f"command: expected one of {', '.join(COMMANDS)}, got {cmd!r}")
    if file_cmd is not None and file_cmd != cmd:
        raise ConfigError(
            f"command: config file says {file_cmd!r} but the CLI was invoked with {cmd!r}")
    if cmd not in SCHEMAS:
        raise ConfigError(f"command {cmd!r} is outside the B200 Gram path (only 'gram', 'bench')")
    schema = SCHEMAS[cmd]
    out = {"command": cmd}
    for k, v in raw.items():
        if k == "command":
            continue
        if k not in schema:
            raise ConfigError(f"unknown config key {k!r} for command {cmd!r}")
        out[k] = schema[k][0](k, v)
    for k, (_, default) in schema.items():
        out.setdefault(k, default)
    for k in _REQUIRED.get(cmd, ()):
        if out[k] is None:
            raise ConfigError(f"{k}: required for command {cmd!r}")
    return out


def load_config(path, command: str = "gram") -> dict:
    try:
        with open(path, "r", encoding="utf-8") as fh:
            text = fh.read()
    except OSError as exc:
        raise ConfigError(f"cannot read config file {path}: {exc}") from exc
    return validate_gram_config(parse_config_text(text), command)


def run_gram(cfg: dict, output: str, precision: str = "fp32") -> None:
    seqs, ids = load_sequences_csv(cfg["input"])
    batch = tabulate(seqs, ids)
    bw = cfg["kernel.static.bandwidth"]
    if bw == "median":
        bw = median_heuristic(batch.data.reshape(-1, batch.data.shape[-1]))
    static = StaticKernelSpec(kind=cfg["kernel.static.kind"], bandwidth=bw,
                              scale=cfg["kernel.static.scale"],
                              degree=cfg["kernel.static.degree"],
                              gamma=cfg["kernel.static.gamma"],
                              alpha=cfg["kernel.static.alpha"])
    kcfg = KernelConfig(static=static, n_levels=cfg["kernel.n_levels"],
                        order=cfg["kernel.order"], difference=cfg["kernel.difference"],
                        normalization=cfg["kernel.normalization"])
    K = sig_kernel_gram(batch, cfg=kcfg, algorithm=cfg["kernel.algorithm"], precision=precision)
    write_matrix_csv(output, K)


def run_bench_cmd(cfg: dict, seed: int, output: str, threads, precision: str = "fp32") -> None:
    """cli.py:197-214: the sweep on the `bench` child stream, then the bench CSV."""
    settings = BenchSettings(
        methods=tuple(cfg["bench.methods"]), n_list=tuple(cfg["bench.n_list"]),
        l_list=tuple(cfg["bench.l_list"]), dq_list=tuple(cfg["bench.dq_list"]),
        m_list=tuple(cfg["bench.m_list"]), dim=cfg["bench.dim"], order=cfg["bench.order"],
        difference=cfg["bench.difference"], static_kind=cfg["kernel.static.kind"],
        bandwidth=cfg["kernel.static.bandwidth"], n_seeds=cfg["bench.n_seeds"],
        compute_mape=cfg["bench.mape"], wall_time=cfg["bench.wall_time"])
    records = run_bench(settings, SeedStream(seed).child("bench"), n_threads=threads or 1,
                        precision=precision)
    write_bench_csv(output, records)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2501_07145_b200",
                                 description="Signature-kernel Gram matrices on B200.")
    ap.add_argument("command", choices=COMMANDS)
    ap.add_argument("--config", required=True)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--output", default=None)
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    args = ap.parse_args(argv)
    try:
        cfg = load_config(args.config, args.command)
        seed = args.seed if args.seed is not None else cfg["seed"]
        if not 0 <= seed < 2 ** 64:
            raise ConfigError(f"seed: expected an unsigned 64-bit integer, got {seed}")
        output = args.output or cfg["output"] or f"sigkern_{args.command}.csv"
        if args.command == "bench":
            run_bench_cmd(cfg, seed, output, args.threads, args.precision)
        else:
            run_gram(cfg, output, args.precision)
    except (ConfigError, ParseError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (SigkernError, ValueError, OSError, NotImplementedError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    return 0
