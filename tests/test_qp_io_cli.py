"""QP text I/O (qp_io.py) and the CLI (cli.py) against reference-written files
and reports (tests/golden/qp_files, made by tests/golden/make_golden.py qp_files)."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, random_case_qp, random_cases

import paper_2003_02547_b200 as pkg
from paper_2003_02547_b200.errors import ParseError, VersionMismatch
from paper_2003_02547_b200.qp_io import qp_dumps, qp_loads, qp_read, qp_write

QPF = GOLDEN / "qp_files"


def test_writer_is_byte_identical_to_reference():
    seed, kw = random_cases()[1]
    assert qp_dumps(random_case_qp(seed, kw)) == (QPF / "rand12.qp").read_text()


def test_read_write_round_trip_is_exact(tmp_path):
    text = (QPF / "rand12.qp").read_text()
    qp = qp_loads(text)
    seed, kw = random_cases()[1]
    ref = random_case_qp(seed, kw)
    for n in range(qp.dim.N + 1):
        for f in ("Q", "S", "R", "q", "r", "idxb", "lb", "ub", "C", "D", "lg", "ug", "idxs",
                  "Zl", "Zu", "zl", "zu", "sl_lb", "su_lb", "maskl", "masku"):
            np.testing.assert_array_equal(qp.get_field(f, n), ref.get_field(f, n))
    qp_write(tmp_path / "x.qp", qp)
    assert (tmp_path / "x.qp").read_text() == text
    assert qp_dumps(qp_read(tmp_path / "x.qp")) == text


@pytest.mark.parametrize("mutate,line,exc", [
    (lambda L: L[:40], None, ParseError),                                  # truncated
    (lambda L: ["mpcqp_qp 2 ocp"] + L[1:], 1, VersionMismatch),
    (lambda L: ["mpcqp_qp 1 dense"] + L[1:], 1, ParseError),
    (lambda L: ["hello"] + L[1:], 1, ParseError),
    (lambda L: L[:2] + ["nx 3 2"] + L[3:], 3, ParseError),                 # count
    (lambda L: L[:10] + ["Qx"] + L[11:], 11, ParseError),                  # field name
    (lambda L: L + ["extra"], None, ParseError),                           # trailing
])
def test_parse_errors_carry_line_numbers(mutate, line, exc):
    lines = (QPF / "rand12.qp").read_text().splitlines()
    with pytest.raises(exc) as ei:
        qp_loads("\n".join(mutate(lines)) + "\n")
    if line is not None:
        assert ei.value.line == line


def test_bad_number_line():
    lines = (QPF / "rand12.qp").read_text().splitlines()
    i = lines.index("Q") + 1
    lines[i] = "1.0 x"
    with pytest.raises(ParseError) as ei:
        qp_loads("\n".join(lines) + "\n")
    assert ei.value.line == i + 1


def _cli(*args, cwd=None):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    return subprocess.run([sys.executable, "-m", "paper_2003_02547_b200", *args],
                          capture_output=True, text=True, env=env, cwd=cwd)


def test_cli_gen_mass_spring_matches_reference(tmp_path):
    r = _cli("gen-mass-spring", "--masses", "3", "--horizon", "6", "--out", str(tmp_path / "m.qp"))
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "m.qp").read_text() == (QPF / "mass3.qp").read_text()


def test_cli_usage_errors_exit_2(tmp_path):
    assert _cli("solve", "--qp", str(tmp_path / "missing.qp")).returncode == 2
    (tmp_path / "bad.qp").write_text("mpcqp_qp 1 tree\n")
    r = _cli("solve", "--qp", str(tmp_path / "bad.qp"))
    assert r.returncode == 2 and "line 1" in r.stderr


def test_cli_solve_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = _cli("solve", "--qp", str(QPF / "mass3.qp"))
    assert r.returncode == 2 and "no CUDA device" in r.stderr


def _report(text):
    head, trace = {}, []
    lines = text.splitlines()
    for i, l in enumerate(lines):
        k, _, v = l.partition(" ")
        if k == "trace":
            head[k] = v
            trace = [list(map(float, x.split())) for x in lines[i + 1:]]
            break
        head[k] = v
    return head, np.array(trace)


@pytest.mark.gpu
@pytest.mark.parametrize("name,extra", [("mass3_balance", []),
                                        ("mass3_speed", ["--mode", "speed", "--tol", "1e-8"]),
                                        ("mass3_partial", ["--path", "partial:2"]),
                                        ("mass3_condense", ["--path", "condense"])])
def test_cli_solve_report_matches_reference(cuda, tmp_path, name, extra):
    import shutil

    shutil.copy(QPF / "mass3.qp", tmp_path / "mass3.qp")
    r = _cli("solve", "--qp", "mass3.qp", *extra, cwd=tmp_path)
    assert r.returncode == 0, r.stderr
    got, gt = _report(r.stdout)
    ref, rt = _report((QPF / f"{name}.report").read_text())
    for k in ("kind", "qp", "solve_path", "mode", "status", "iterations", "trace"):
        assert got[k] == ref[k], k
    fl = int(got["flops"]) - int(ref["flops"])
    if "speed" in extra:
        assert fl == 0
    else:  # balance: the number of refinement solves may differ (tests/modes_common.py)
        assert abs(fl) <= 0.1 * int(ref["flops"])
    for k in ("res_g", "res_b", "res_d", "res_m", "mu"):
        assert abs(float(got[k]) - float(ref[k])) <= 1e-8 * max(1.0, abs(float(ref[k])))
    np.testing.assert_allclose(gt[:, :5], rt[:, :5], rtol=1e-6, atol=1e-12)
