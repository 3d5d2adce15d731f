"""Text formats: instance files, solution line, LP export
and the run artifacts of ``dmmv solve``, against the reference's own test
cases (``/root/reference/pkg/tests/test_io.py``) and golden text made by the
unmodified reference (``tests/golden/make_golden_formats.py``).

CPU tests cover the host-side formats; the ``gpu`` test solves each golden
instance through the CUDA path and checks report.txt / trace.csv /
solution.txt byte for byte against the reference CLI's files.
"""

import io
import json
import os

import numpy as np
import pytest

import paper_2508_13437_b200 as P

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "formats.json")))["cases"]
BASE = "2 2 2\n0.0 1.0\n0.5 -1.5\n1.0 -2.0\n0.0 3.0\n"


def _base(init=None):
    return P.Instance(np.array([[1.0, -2.0], [0.0, 3.0]]), np.array([0.5, -1.5]),
                      P.ValueSet([0.0, 1.0]), continuous_init=init)


@pytest.mark.parametrize("k", range(len(GOLDEN)))
def test_golden_instance_text_round_trips_byte_identical(k):
    text = GOLDEN[k]["instance"]
    inst = P.read_instance(io.StringIO(text))
    assert P.instance_to_text(inst) == text
    buf = io.StringIO()
    P.write_instance(inst, buf)
    assert buf.getvalue() == text


@pytest.mark.parametrize("k", range(len(GOLDEN)))
def test_golden_lp_export_matches_reference(k):
    inst = P.read_instance(io.StringIO(GOLDEN[k]["instance"]))
    buf = io.StringIO()
    P.export_lp(inst, buf)
    assert buf.getvalue() == GOLDEN[k]["lp"]
    assert all(len(ln) <= 72 for ln in buf.getvalue().splitlines() if len(ln.split()) > 1)


def test_layout_and_init_line(tmp_path):
    path = tmp_path / "inst.txt"
    P.write_instance(_base(), path)
    assert path.read_text() == BASE
    assert P.instance_to_text(_base(np.array([0.25, 0.75]))) == BASE + "init 0.25 0.75\n"


def test_blank_lines_and_file_objects():
    inst = P.read_instance(io.StringIO("\n2 2 2\n\n0.0 1.0\n0.5 -1.5\n\n\n1.0 -2.0\n0.0 3.0\n\n"))
    assert (inst.m, inst.n, inst.continuous_init) == (2, 2, None)


@pytest.mark.parametrize("text, pattern, line, token", [
    ("1 2 2\n0.0 1.0\n", "line 3: missing b line", 3, None),
    ("2 2\n", r"3 integers.*found 2 tokens", 1, None),
    ("2 x 2\n", "bad integer 'x' in header", 1, 2),
    ("2 0 2\n", "must be positive, found 0", 1, 2),
    ("\n\n2 nope 2\n", "bad integer", 3, 2),
    ("1 1 3\n0.0 1.0\n", "expected 3 values for levels, found 2", 2, None),
    ("1 1 3\n0.0 abc 1.0\n", "bad number 'abc' in levels", 2, 2),
    ("1 1 2\n1.0 0.0\n0.5\n1.0\n", "strictly increasing", 2, None),
    ("2 2 2\n0.0 1.0\n0.5 -1.5\n1.0 -2.0\n0.0 oops\n", "bad number 'oops' in row 2 of A", 5, 2),
    ("2 2 2\n0.0 1.0\n0.5 -1.5\n1.0 -2.0\n0.0\n", "expected 2 values for row 2 of A", 5, None),
    (BASE + "foo bar\n", "unexpected trailing content 'foo'", 6, 1),
    (BASE + "init 0.5\n", "expected 2 values for init", 6, None),
    (BASE + "init 0.5 0.5\n0.1\n", "after the init line", 7, None),
])
def test_parse_diagnostics(text, pattern, line, token):
    with pytest.raises(P.InstanceParseError, match=pattern) as exc:
        P.read_instance(io.StringIO(text))
    assert exc.value.line == line and exc.value.token == token
    assert isinstance(exc.value, ValueError)


def test_solution_line_is_init_compatible(tmp_path):
    inst = _base()
    sol = P.Solution.from_indices(inst, [1, 0])
    path = tmp_path / "sol.txt"
    P.write_solution(sol, inst, path)
    assert path.read_text() == "1.0 0.0\n"
    back = P.read_instance(io.StringIO(BASE + "init " + path.read_text()))
    np.testing.assert_array_equal(back.continuous_init, [1.0, 0.0])


def test_lp_exact_text():
    buf = io.StringIO()
    P.export_lp(_base(), buf)
    assert buf.getvalue() == (
        "Minimize\n obj: t\nSubject To\n"
        " up_0:\n  + 1.0 z_0_1 - 2.0 z_1_1 - t <= 0.5\n"
        " lo_0:\n  + 1.0 z_0_1 - 2.0 z_1_1 + t >= 0.5\n"
        " up_1:\n  + 3.0 z_1_1 - t <= -1.5\n"
        " lo_1:\n  + 3.0 z_1_1 + t >= -1.5\n"
        " sel_0:\n  + z_0_0 + z_0_1 = 1\n"
        " sel_1:\n  + z_1_0 + z_1_1 = 1\n"
        "Bounds\n t >= 0\nBinaries\n  z_0_0 z_0_1 z_1_0 z_1_1\nEnd\n")


@pytest.mark.gpu
@pytest.mark.parametrize("k", [k for k, c in enumerate(GOLDEN) if "trace" in c])
def test_run_artifacts_match_reference_cli(tmp_path, k):
    """``dmmv solve --iters I --seed S`` on the golden instance: the CUDA path's
    report.txt (minus wall time / instance path), trace.csv and solution.txt
    equal the reference CLI's byte for byte."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    rec = GOLDEN[k]
    inst = P.read_instance(io.StringIO(rec["instance"]))
    cfg = P.SolverConfig(max_iters=rec["iters"], seed=rec["seed"])
    rep = P.solve(inst, cfg)
    paths = P.write_run_artifacts(inst, cfg, rep, tmp_path / "run", "inst.txt")
    lines = [ln for ln in paths.report.read_text().splitlines()
             if not ln.startswith(("wall_time_s", "instance:"))]
    ref = [ln for ln in rec["report"] if not ln.startswith("solver_version")]
    assert [ln for ln in lines if not ln.startswith("solver_version")] == ref
    assert paths.trace.read_text() == rec["trace"]
    assert paths.solution.read_text() == rec["solution"]
