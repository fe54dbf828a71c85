"""Versioned text formats of the reference (io.cpp) and the synthetic trace
generator (trace_gen.cpp) — the data formats either side of the hot path
(SURVEY.md 8(f) rows 3-4): routing traces in, co-activation matrices and
placements between the profiling and placement steps.

Byte-compatible with the reference in both directions: writers produce the
reference's bytes (doubles in std::to_chars shortest form, `report.format_double`),
readers accept exactly what std::from_chars / std::getline / operator>> accept
and raise `DataError` with the reference's `line N: ...` messages.  The
generator runs in the native library (`occ_gen_trace`, std::mt19937_64).
"""
from __future__ import annotations

import ctypes as C
import math
import re
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from . import api
from .report import format_double

TRACE_HEADER = "#moesim-trace v1"          # io.cpp:15
MATRIX_HEADER = "#moesim-matrix v1"        # io.cpp:16
PLACEMENT_HEADER = "#moesim-placement v1"  # io.cpp:17


DataError = api.DataError
UsageError = api.UsageError


# ---------------------------------------------------------------- lexing --
_WS = re.compile(r"[ \t\n\v\f\r]+")
_INT = re.compile(r"-?[0-9]+")
_FLOAT = re.compile(r"-?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?")
_SPECIAL = re.compile(r"-?(?:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?)", re.IGNORECASE)


def _split_ws(line: str) -> List[str]:
    """operator>> over an istringstream (io.cpp:20-26)."""
    return [t for t in _WS.split(line) if t]


def _lines(text: str) -> List[str]:
    """std::getline: split on '\\n'; a final newline does not start a line."""
    parts = text.split("\n")
    if parts and parts[-1] == "":
        parts.pop()
    return parts


def _bad(line_no: int, what: str):
    raise DataError(f"line {line_no}: {what}")


def parse_int(s: str, line_no: int) -> int:
    """std::from_chars(long long) over the whole token (io.cpp:32-39)."""
    if not _INT.fullmatch(s) or not -(1 << 63) <= int(s) < (1 << 63):
        _bad(line_no, f"expected integer, got '{s}'")
    return int(s)


def _to_int32(v: int) -> int:
    """static_cast<int>(long long): two's-complement wrap."""
    return C.c_int32(v).value


def parse_double(s: str, line_no: int) -> float:
    """std::from_chars(double), general format, over the whole token
    (io.cpp:62-69): no leading '+' or whitespace; out-of-range magnitudes
    are errors."""
    if _SPECIAL.fullmatch(s):
        neg = s.startswith("-")
        body = s[1:] if neg else s
        v = float("nan") if body[:3].lower() == "nan" else float("inf")
        return -v if neg else v
    if not _FLOAT.fullmatch(s):
        _bad(line_no, f"expected number, got '{s}'")
    v = float(s)
    if math.isinf(v):
        _bad(line_no, f"expected number, got '{s}'")
    if v == 0.0 and re.search(r"[1-9]", s.split("e")[0].split("E")[0]):
        _bad(line_no, f"expected number, got '{s}'")  # underflow to zero
    return v


def _expect_header(lines: List[str], header: str):
    """io.cpp:43-52: the header line, then the fields line."""
    if not lines:
        raise DataError("line 1: empty input")
    if lines[0] != header:
        _bad(1, f"expected header '{header}'")
    if len(lines) < 2:
        _bad(2, "missing header fields")
    return lines[1]


# ----------------------------------------------------------------- trace --
@dataclass
class TraceFile:
    """io.hpp:17-22: routed-token trace (ids in descending score order)."""
    num_experts: int
    top_k: int
    ids: np.ndarray                      # int32 [n, k]
    weights: np.ndarray                  # float64 [n, k]
    tag: str = ""

    @property
    def num_tokens(self) -> int:
        return int(self.ids.shape[0])


def write_trace(trace: TraceFile) -> str:
    """io.cpp:71-86."""
    n, k = trace.num_tokens, trace.top_k
    out = [TRACE_HEADER + "\n",
           f"experts={trace.num_experts} topk={k} tokens={n}" + (f" tag={trace.tag}" if trace.tag else "") + "\n"]
    ids = np.asarray(trace.ids).reshape(n, k).tolist()
    ws = np.asarray(trace.weights, dtype=np.float64).reshape(n, k).tolist()
    for t in range(n):
        out.append(" ".join(map(str, ids[t])) + " " + " ".join(format_double(w) for w in ws[t]) + "\n")
    return "".join(out)


def _validate_routing(ids, ws, n, k, num_experts):
    """RoutingOutcome::validate (routing.cpp:11-31), re-raised as DataError."""
    for t in range(n):
        row = ids[t]
        for j in range(k):
            if row[j] < 0 or row[j] >= num_experts:
                raise DataError(f"trace file: routing: expert id out of range at token {t}")
            if ws[t][j] <= 0.0:  # NaN passes, as in the reference
                raise DataError(f"trace file: routing: non-positive weight at token {t}")
            if row[j] in row[:j]:
                raise DataError(f"trace file: routing: duplicate expert id at token {t}")


def read_trace(text: str) -> TraceFile:
    """io.cpp:88-137."""
    lines = _lines(text)
    fields = _expect_header(lines, TRACE_HEADER)
    line_no = 2
    num_experts = top_k = 0
    tokens = -1
    tag = ""
    for f in _split_ws(fields):
        eq = f.find("=")
        if eq < 0:
            _bad(line_no, f"malformed header field '{f}'")
        key, val = f[:eq], f[eq + 1:]
        if key == "experts":
            num_experts = _to_int32(parse_int(val, line_no))
        elif key == "topk":
            top_k = _to_int32(parse_int(val, line_no))
        elif key == "tokens":
            tokens = _to_int32(parse_int(val, line_no))
        elif key == "tag":
            tag = val
        else:
            _bad(line_no, f"unknown header field '{key}'")
    if num_experts < 1 or top_k < 1 or tokens < 0:
        _bad(line_no, "incomplete trace header")
    ids: List[List[int]] = []
    ws: List[List[float]] = []
    for line in lines[2:]:
        line_no += 1
        if line == "":
            continue
        parts = _split_ws(line)
        if len(parts) != 2 * top_k:
            _bad(line_no, f"record needs {2 * top_k} fields, got {len(parts)}")
        row = []
        for j in range(top_k):
            v = parse_int(parts[j], line_no)
            if v < 0 or v >= num_experts:
                _bad(line_no, "expert id out of range")
            row.append(v)
        ids.append(row)
        ws.append([parse_double(parts[top_k + j], line_no) for j in range(top_k)])
    if len(ids) != tokens:
        raise DataError(f"trace declares {tokens} tokens but has {len(ids)} records")
    _validate_routing(ids, ws, tokens, top_k, num_experts)
    return TraceFile(num_experts, top_k, np.array(ids, dtype=np.int32).reshape(tokens, top_k),
                     np.array(ws, dtype=np.float64).reshape(tokens, top_k), tag)


# ---------------------------------------------------------------- matrix --
def write_matrix(m) -> str:
    """io.cpp:139-148."""
    m = np.asarray(m, dtype=np.float64)
    rows, cols = m.shape
    out = [MATRIX_HEADER + "\n", f"{rows} {cols}\n"]
    for r in m.tolist():
        out.append(" ".join(format_double(v) for v in r) + "\n")
    return "".join(out)


def read_matrix(text: str) -> np.ndarray:
    """io.cpp:150-166."""
    lines = _lines(text)
    shape = _split_ws(_expect_header(lines, MATRIX_HEADER))
    line_no = 2
    if len(shape) != 2:
        _bad(line_no, "expected 'rows cols'")
    rows, cols = _to_int32(parse_int(shape[0], line_no)), _to_int32(parse_int(shape[1], line_no))
    if rows < 0 or cols < 0:
        raise DataError(f"line {line_no}: negative matrix shape")  # the reference would fail to allocate
    m = np.zeros((rows, cols), np.float64)
    for i in range(rows):
        if 2 + i >= len(lines):
            _bad(line_no + 1, "missing matrix row")
        line_no += 1
        parts = _split_ws(lines[2 + i])
        if len(parts) != cols:
            _bad(line_no, "wrong column count")
        m[i] = [parse_double(p, line_no) for p in parts]
    return m


# ------------------------------------------------------------- placement --
def write_placement(p: "api.Placement") -> str:
    """io.cpp:168-178."""
    out = [PLACEMENT_HEADER + "\n", f"devices={len(p.devices)}\n"]
    for dev in p.devices:
        out.append(" ".join(str(int(e)) for e in dev) + "\n")
    return "".join(out)


def validate_placement(devices: Sequence[Sequence[int]], expected_experts: int = -1):
    """Placement::validate (placement.cpp:32-45) with its PlacementError texts."""
    if not devices:
        raise api.PlacementError("placement: no devices")
    n = sum(len(d) for d in devices)
    if expected_experts >= 0 and n != expected_experts:
        raise api.PlacementError(f"placement: covers {n} experts, expected {expected_experts}")
    if n % len(devices) or any(len(d) != n // len(devices) for d in devices):
        raise api.PlacementError("placement: uneven device lists")
    seen = [False] * n
    for d in devices:
        for e in d:
            if e < 0 or e >= n or seen[e]:
                raise api.PlacementError(f"placement: device lists are not a partition of [0, {n})")
            seen[e] = True


def read_placement(text: str) -> "api.Placement":
    """io.cpp:180-204."""
    lines = _lines(text)
    parts = _split_ws(_expect_header(lines, PLACEMENT_HEADER))
    line_no = 2
    if len(parts) != 1 or not parts[0].startswith("devices="):
        _bad(line_no, "expected 'devices=N'")
    nd = _to_int32(parse_int(parts[0][8:], line_no))
    devices = []
    for d in range(nd):
        if 2 + d >= len(lines):
            _bad(line_no + 1, "missing device list")
        line_no += 1
        devices.append([_to_int32(parse_int(t, line_no)) for t in _split_ws(lines[2 + d])])
    try:
        validate_placement(devices)
    except api.PlacementError as e:
        raise DataError(f"placement file: {e}") from None
    return api.Placement(devices)


# ------------------------------------------------------ trace generation --
DISTS = {"uniform": 0, "zipf": 1, "blocks": 2}


class _Spec(C.Structure):
    _fields_ = [("dist", C.c_int), ("num_experts", C.c_int), ("top_k", C.c_int), ("num_tokens", C.c_int),
                ("alpha", C.c_double), ("num_blocks", C.c_int), ("p_in", C.c_double)]


@dataclass
class TraceSpec:
    """trace_gen.hpp:12-33."""
    dist: str = "uniform"
    num_experts: int = 0
    top_k: int = 0
    num_tokens: int = 0
    alpha: float = 0.0
    num_blocks: int = 1
    p_in: float = 0.9
    tag: str = ""


def gen_trace(spec: TraceSpec, seed: int) -> TraceFile:
    """gen_trace (trace_gen.cpp:56-122) in the native library; identical to the
    reference's trace for the same spec and seed."""
    if spec.dist not in DISTS:
        raise UsageError(f"unknown distribution '{spec.dist}'")
    lib = api.lib()
    n, k = max(spec.num_tokens, 0), max(spec.top_k, 0)
    ids = np.empty((n, k), np.int32)
    ws = np.empty((n, k), np.float64)
    cs = _Spec(DISTS[spec.dist], spec.num_experts, spec.top_k, spec.num_tokens, spec.alpha, spec.num_blocks,
               spec.p_in)
    rc = lib.occ_gen_trace(C.byref(cs), C.c_uint64(seed & (2 ** 64 - 1)), ids.ctypes.data_as(C.c_void_p),
                           ws.ctypes.data_as(C.c_void_p))
    if rc:
        raise UsageError(lib.occ_last_error().decode())
    return TraceFile(spec.num_experts, spec.top_k, ids, ws, spec.tag)


class Rng:
    """rng.hpp:12-38 (std::mt19937_64 + the reference's draws), native."""

    def __init__(self, seed: int):
        self._lib = api.lib()
        self._h = C.c_void_p()
        api._check(self._lib.occ_rng_create(C.c_uint64(seed & (2 ** 64 - 1)), C.byref(self._h)), "rng")

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.occ_rng_destroy(self._h)
            self._h = None

    def next(self) -> int:
        return int(self._lib.occ_rng_next(self._h))

    def random_matrix(self, rows: int, cols: int, single: bool = True) -> np.ndarray:
        """random_matrix (core.cpp:54-58)."""
        out = np.empty((rows, cols), np.float64)
        api._check(self._lib.occ_rng_matrix(self._h, rows, cols, int(single), out.ctypes.data_as(C.c_void_p)),
                   "random_matrix")
        return out
