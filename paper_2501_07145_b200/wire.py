"""Wire formats around the Gram path (host side, not on the device path).

* sequence CSV `seq_id,step,c0,..` -> ragged sequences (load_sequences_csv,
  sequences.py:186-245), and the tabulation that makes a uniform batch of them
  (tabulate, preprocessing.py:97-128: channel-wise linear fill of missing
  cells, piecewise-linear resampling to the longest length);
* headerless matrix CSV with round-trip float formatting (write_matrix_csv,
  sequences.py:140-155) — the output of `gram`, byte-identical to the
  reference's writer for the same matrix.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import ParseError
from .sequences import SequenceBatch

__all__ = ["format_value", "write_matrix_csv", "read_matrix_csv", "load_sequences_csv",
           "write_sequences_csv", "tabulate"]


def format_value(v) -> str:
    """Integral values print as integers, everything else as repr (sequences.py:140-144)."""
    f = float(v)
    if math.isfinite(f) and f == int(f) and abs(f) < 1e16:
        return str(int(f))
    return repr(f)


def write_matrix_csv(path, matrix) -> None:
    matrix = np.asarray(matrix)
    if matrix.ndim != 2:
        raise ValueError(f"matrix must be 2-D, got shape {matrix.shape}")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        for row in matrix:
            fh.write(",".join(format_value(v) for v in row) + "\n")


def read_matrix_csv(path) -> np.ndarray:
    with open(path, "r", encoding="utf-8") as fh:
        rows = [ln for ln in fh.read().splitlines() if ln.strip()]
    return np.array([[float(c) for c in r.split(",")] for r in rows], dtype=np.float64)


def _parse_int(cell: str, what: str, line: int) -> int:
    try:
        v = int(cell)
    except ValueError:
        raise ParseError(f"{what} must be an integer, got {cell!r}", line=line) from None
    if v < 0:
        raise ParseError(f"{what} must be non-negative, got {v}", line=line)
    return v


def load_sequences_csv(path):
    """-> (list of (L_i, d) arrays with NaN for empty cells, ids), ordered by seq_id,
    rows ordered by step; malformed rows raise ParseError with the line number."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise ParseError("empty file", line=1)
    header = [h.strip() for h in lines[0].split(",")]
    if len(header) < 3 or header[0] != "seq_id" or header[1] != "step":
        raise ParseError(f"header must be 'seq_id,step,c0,...', got {lines[0]!r}", line=1)
    d = len(header) - 2
    rows: dict[int, list] = {}
    for lineno, raw in enumerate(lines[1:], start=2):
        if not raw.strip():
            continue
        cells = raw.split(",")
        if len(cells) != d + 2:
            raise ParseError(f"expected {d + 2} fields, got {len(cells)}", line=lineno)
        sid = _parse_int(cells[0].strip(), "seq_id", lineno)
        step = _parse_int(cells[1].strip(), "step", lineno)
        vals = np.empty(d)
        for j, cell in enumerate(cells[2:]):
            cell = cell.strip()
            if not cell:
                vals[j] = np.nan
                continue
            try:
                vals[j] = float(cell)
            except ValueError:
                raise ParseError(f"channel c{j} must be numeric or empty, got {cell!r}",
                                 line=lineno) from None
        rows.setdefault(sid, []).append((step, lineno, vals))
    if not rows:
        raise ParseError("file contains a header but no data rows", line=2)
    seqs, ids = [], []
    for sid in sorted(rows):
        ent = sorted(rows[sid], key=lambda e: e[0])
        for a, b in zip(ent, ent[1:]):
            if a[0] == b[0]:
                raise ParseError(f"duplicate step {b[0]} for seq_id {sid}", line=b[1])
        seqs.append(np.stack([e[2] for e in ent]))
        ids.append(sid)
    return seqs, ids


def write_sequences_csv(path, batch: SequenceBatch) -> None:
    d = batch.data.shape[2]
    order = np.argsort(np.asarray(batch.ids), kind="stable")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("seq_id,step," + ",".join(f"c{j}" for j in range(d)) + "\n")
        for i in order:
            for step, pt in enumerate(batch.data[i]):
                cells = ["" if math.isnan(v) else format_value(v) for v in pt]
                fh.write(f"{int(batch.ids[i])},{step}," + ",".join(cells) + "\n")


def _fill_missing(x: np.ndarray, sid: int) -> np.ndarray:
    if not np.isnan(x).any():
        return x
    x = x.copy()
    grid = np.arange(x.shape[0], dtype=np.float64)
    for c in range(x.shape[1]):
        obs = ~np.isnan(x[:, c])
        k = int(obs.sum())
        if k < 2:
            raise ValueError(f"sequence {sid}: channel {c} has {k} observed value(s); "
                             f"tabulation needs at least 2 per channel")
        if k < x.shape[0]:
            x[:, c] = np.interp(grid, grid[obs], x[obs, c])
    return x


def _resample(x: np.ndarray, n: int) -> np.ndarray:
    L = x.shape[0]
    if n == L:
        return x.copy()
    if n == 1 or L == 1:
        return np.repeat(x[:1], n, axis=0)
    u = np.arange(n) * (L - 1) / (n - 1)
    i = np.minimum(np.floor(u).astype(np.int64), L - 2)
    f = u - i
    out = x[i] + f[:, None] * (x[i + 1] - x[i])
    on_grid = f == 0.0  # grid points on a source index are copied bitwise
    if on_grid.any():
        out[on_grid] = x[i[on_grid]]
    return out


def tabulate(seqs, ids=None, max_len: int | None = None) -> SequenceBatch:
    arrays = [np.asarray(s, dtype=np.float64) for s in seqs]
    ids = np.arange(len(arrays), dtype=np.int64) if ids is None else np.asarray(ids, np.int64)
    if not arrays:
        raise ValueError("tabulate needs at least one sequence")
    dims = {a.shape[1] for a in arrays}
    if len(dims) != 1:
        raise ValueError(f"sequences disagree on channel count: {sorted(dims)}")
    target = max(a.shape[0] for a in arrays)
    if max_len is not None:
        if max_len < 1:
            raise ValueError(f"max_len must be positive, got {max_len}")
        target = min(target, int(max_len))
    filled = [_fill_missing(a, int(i)) for a, i in zip(arrays, ids)]
    for a, i in zip(filled, ids):
        if a.shape[0] < 2 and a.shape[1] > 0:
            raise ValueError(f"sequence {int(i)}: channel 0 has {a.shape[0]} observed value(s); "
                             f"tabulation needs at least 2 per channel")
    return SequenceBatch(np.stack([_resample(a, target) for a in filled]), ids)
