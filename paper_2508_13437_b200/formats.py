"""Instance text format, solution line, LP export and run artifacts.

SURVEY.md §8f-4: the data formats on either side of the ``solve`` path.
Host-side by nature (text in, text out); the arrays they produce or consume
are what the device path works on.  Byte-for-byte the reference's formats:

* instance file -- ``/root/reference/pkg/src/dmmv/io.py:1-12`` (layout),
  ``io.py:44-59`` (writer), ``io.py:101-151`` (parser and its diagnostics);
* solution line -- ``io.py:154-162``;
* LP export -- ``io.py:165-229`` (72-column wrapping, zero coefficients
  skipped, selector binaries);
* run artifacts ``report.txt`` / ``trace.csv`` / ``solution.txt`` --
  ``cli.py:99-140`` (``cmd_solve``).

Floats are written with ``repr`` (shortest round-trip decimal), so
write -> read -> write is the identity on the text.
"""

from __future__ import annotations

import io as _stdio
from dataclasses import dataclass
from pathlib import Path
from typing import IO, Iterable, Iterator

import numpy as np

from .core import Instance, Solution, ValueSet

LP_LINE_WIDTH = 72  # io.py:165


class InstanceParseError(ValueError):
    """A parse failure at a 1-based line (and optional token) position.

    Message layout ``"line L[, token T]: what"`` as ``io.py:26-33``.
    """

    def __init__(self, message: str, line: int, token: int | None = None) -> None:
        self.line = line
        self.token = token
        loc = f"line {line}" if token is None else f"line {line}, token {token}"
        super().__init__(f"{loc}: {message}")


def format_values(vec: Iterable[float]) -> str:
    """Space-separated shortest round-trip decimals (``io.py:36-41``)."""
    return " ".join(repr(float(x)) for x in vec)


class _Sink:
    """Context manager: a path is opened for writing and closed, a stream is
    borrowed as is."""

    def __init__(self, target) -> None:
        self._own = isinstance(target, (str, Path))
        self._target = target

    def __enter__(self) -> IO[str]:
        self._fh = open(self._target, "w") if self._own else self._target
        return self._fh

    def __exit__(self, *exc) -> None:
        if self._own:
            self._fh.close()


# ---------------------------------------------------------------- instance


def _instance_lines(inst: Instance) -> Iterator[str]:
    yield f"{inst.m} {inst.n} {len(inst.values)}"
    yield format_values(inst.values.levels)
    yield format_values(inst.b)
    for row in inst.A:
        yield format_values(row)
    if inst.continuous_init is not None:
        yield "init " + format_values(inst.continuous_init)


def write_instance(inst: Instance, target: str | Path | IO[str]) -> None:
    """Write ``inst`` in the text format (``io.py:44-59``)."""
    with _Sink(target) as fh:
        for line in _instance_lines(inst):
            fh.write(line + "\n")


def instance_to_text(inst: Instance) -> str:
    return "".join(line + "\n" for line in _instance_lines(inst))


class _TokenLines:
    """The non-blank lines of a text, tokenised, with 1-based line numbers
    counting blank lines too (``io.py:62-84``)."""

    def __init__(self, text: str) -> None:
        self._rows = [(no, ln.split()) for no, ln in enumerate(text.splitlines(), 1)
                      if ln.strip()]
        self._at = 0

    def take(self, what: str) -> tuple[int, list[str]]:
        if self._at == len(self._rows):
            after = self._rows[-1][0] if self._rows else 1
            raise InstanceParseError(f"missing {what}", after + 1)
        self._at += 1
        return self._rows[self._at - 1]

    @property
    def done(self) -> bool:
        return self._at == len(self._rows)


def _parse_floats(tokens: list[str], line: int, count: int, what: str) -> np.ndarray:
    """``io.py:87-98``: exact count, each token a Python float."""
    if len(tokens) != count:
        raise InstanceParseError(
            f"expected {count} values for {what}, found {len(tokens)}", line)
    vals = np.empty(count)
    for pos, tok in enumerate(tokens, 1):
        try:
            vals[pos - 1] = float(tok)
        except ValueError:
            raise InstanceParseError(f"bad number {tok!r} in {what}", line,
                                     token=pos) from None
    return vals


def _parse_header(tokens: list[str], line: int) -> tuple[int, int, int]:
    if len(tokens) != 3:
        raise InstanceParseError(
            f"header must read 'm n v' (3 integers), found {len(tokens)} tokens", line)
    dims = []
    for pos, tok in enumerate(tokens, 1):
        try:
            d = int(tok)
        except ValueError:
            raise InstanceParseError(f"bad integer {tok!r} in header", line,
                                     token=pos) from None
        if d < 1:
            raise InstanceParseError(
                f"header dimensions must be positive, found {d}", line, token=pos)
        dims.append(d)
    return dims[0], dims[1], dims[2]


def read_instance(source: str | Path | IO[str]) -> Instance:
    """Parse the text format into an :class:`Instance` (``io.py:101-151``).

    Every diagnostic is an :class:`InstanceParseError` (a ``ValueError``)
    naming the line, and the token where one is at fault.
    """
    text = Path(source).read_text() if isinstance(source, (str, Path)) else source.read()
    src = _TokenLines(text)

    line, toks = src.take("header line 'm n v'")
    m, n, nlev = _parse_header(toks, line)

    line, toks = src.take("levels line")
    levels = _parse_floats(toks, line, nlev, "levels")
    if nlev > 1 and not bool(np.all(levels[1:] > levels[:-1])):
        raise InstanceParseError("levels must be strictly increasing", line)

    line, toks = src.take("b line")
    b = _parse_floats(toks, line, m, "b")

    A = np.empty((m, n))
    for r in range(1, m + 1):
        line, toks = src.take(f"row {r} of A")
        A[r - 1] = _parse_floats(toks, line, n, f"row {r} of A")

    init = None
    if not src.done:
        line, toks = src.take("trailing content")
        if toks[0] != "init":
            raise InstanceParseError(
                f"unexpected trailing content {toks[0]!r}; only an 'init' line may "
                "follow A", line, token=1)
        init = _parse_floats(toks[1:], line, n, "init")
        if not src.done:
            line, _ = src.take("trailing content")
            raise InstanceParseError("unexpected content after the init line", line)

    return Instance(A, b, ValueSet(levels), continuous_init=init)


def write_solution(sol: Solution, inst: Instance, target: str | Path | IO[str]) -> None:
    """One line with the solution's level values; it can be pasted after
    ``init`` in an instance file (``io.py:154-162``)."""
    with _Sink(target) as fh:
        fh.write(format_values(inst.values.levels[np.asarray(sol.idx)]) + "\n")


# ---------------------------------------------------------------- LP export


def _wrap(fh: IO[str], terms: list[str], cont: str = "   ") -> None:
    """Greedy wrap at LP_LINE_WIDTH: first line starts with one space, later
    lines with ``cont``; each term is preceded by a space (``io.py:168-176``)."""
    buf = " "
    for term in terms:
        if buf.strip() and len(buf) + 1 + len(term) > LP_LINE_WIDTH:
            fh.write(buf + "\n")
            buf = cont
        buf = f"{buf} {term}"
    if buf.strip():
        fh.write(buf + "\n")


def export_lp(inst: Instance, target: str | Path | IO[str]) -> None:
    """Exact MILP reformulation in LP format (``io.py:190-229``).

    ``min t`` s.t. ``±(Σ_j Σ_v a_kj·lv_v·z_j_v − b_k) ≤ t`` per row and
    ``Σ_v z_j_v = 1`` per variable, ``z`` binary.
    """
    lv = inst.values.levels
    nlev = lv.size
    zname = [f"z_{j}_{v}" for j in range(inst.n) for v in range(nlev)]
    with _Sink(target) as fh:
        fh.write("Minimize\n obj: t\nSubject To\n")
        for k in range(inst.m):
            coef = (inst.A[k][:, None] * lv[None, :]).reshape(-1)
            terms = [f"{'-' if c < 0 else '+'} {abs(float(c))!r} {zname[q]}"
                     for q, c in enumerate(coef) if c != 0]
            rhs = repr(float(inst.b[k]))
            fh.write(f" up_{k}:\n")
            _wrap(fh, terms + ["- t", "<=", rhs])
            fh.write(f" lo_{k}:\n")
            _wrap(fh, terms + ["+ t", ">=", rhs])
        for j in range(inst.n):
            fh.write(f" sel_{j}:\n")
            _wrap(fh, ["+ " + zname[j * nlev + v] for v in range(nlev)] + ["=", "1"])
        fh.write("Bounds\n t >= 0\nBinaries\n")
        _wrap(fh, zname, cont=" ")
        fh.write("End\n")


# ---------------------------------------------------------------- run artifacts


@dataclass(frozen=True)
class RunArtifacts:
    """The files one solve run writes (``cli.py:45-50``)."""

    report: Path
    trace: Path
    solution: Path


def report_lines(inst: Instance, cfg, report, instance_name: str,
                 solver_version: str) -> list[str]:
    """``report.txt`` body, key order and formatting of ``cli.py:109-127``."""
    return [
        f"solver_version: {solver_version}",
        f"instance: {instance_name}",
        f"m: {inst.m}",
        f"n: {inst.n}",
        f"levels: {len(inst.values)}",
        f"seed: {cfg.seed}",
        f"iters_requested: {cfg.max_iters}",
        f"time_limit: {cfg.time_limit}",
        f"destroy_rate: {cfg.destroy_rate}",
        f"alpha: {cfg.alpha}",
        f"k_eps: {cfg.k_eps}",
        f"max_candidates: {cfg.max_candidates}",
        f"workers: {cfg.workers}",
        f"initial_objective: {report.initial_objective!r}",
        f"best_objective: {report.best.objective!r}",
        f"iterations_run: {report.iterations}",
        f"wall_time_s: {report.wall_time:.3f}",
    ]


def trace_csv(report) -> str:
    """``trace.csv`` text (``cli.py:129-135``)."""
    out = _stdio.StringIO()
    out.write("iter,current_t,best_t,op_pair,accepted\n")
    for e in report.trace:
        out.write(f"{e.iteration},{e.current_t!r},{e.best_t!r},{e.op_pair},"
                  f"{int(e.accepted)}\n")
    return out.getvalue()


def write_run_artifacts(inst: Instance, cfg, report, outdir: str | Path,
                        instance_name: str, solver_version: str | None = None
                        ) -> RunArtifacts:
    """Write ``report.txt``, ``trace.csv`` and ``solution.txt`` under
    ``outdir`` exactly as ``dmmv solve`` does (``cli.py:99-140``)."""
    if solver_version is None:
        from . import __version__ as solver_version
    out = Path(outdir)
    out.mkdir(parents=True, exist_ok=True)
    paths = RunArtifacts(out / "report.txt", out / "trace.csv", out / "solution.txt")
    paths.report.write_text(
        "\n".join(report_lines(inst, cfg, report, instance_name, solver_version)) + "\n")
    paths.trace.write_text(trace_csv(report))
    write_solution(report.best, inst, paths.solution)
    return paths
