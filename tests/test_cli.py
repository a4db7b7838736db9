"""The `cluster` front-end (SPEC.md [MODULE] cli, cmd_cluster) --
paper_2006_06743_b200/bin/sngb_cluster over the C++ mirror.

CPU: flag errors exit 2 with usage text before any computation, I/O errors
exit 3.  GPU: the SPEC example (4-point line, eps=1, min-pts=1, rate=1 ->
labels 0 0 1 1, k=2) and a synthetic set against the oracle."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2006_06743_b200 as sng
from paper_2006_06743_b200 import io as sio
from paper_2006_06743_b200.build import CLI, build_cli


@pytest.fixture(scope="module")
def cli():
    build_cli()
    return CLI


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True)


def _line4(tmp_path):
    p = tmp_path / "line.sngd"
    sio.save_binary(sng.Dataset(np.array([[0.0], [0.5], [10.0], [10.5]])), str(p))
    return p


def test_flag_errors_exit_2_with_usage(cli, tmp_path):
    p = _line4(tmp_path)
    r = run(cli, "--input", p, "--min-pts", 1)  # missing --eps
    assert r.returncode == 2 and "usage:" in r.stderr and "missing --eps" in r.stderr
    r = run(cli, "--input", p, "--eps", 1, "--min-pts", 1, "--rate", 1.5)
    assert r.returncode == 2 and "rate must lie in (0, 1]" in r.stderr
    r = run(cli, "--input", p, "--eps", 0, "--min-pts", 1)
    assert r.returncode == 2 and "eps must be > 0" in r.stderr
    r = run(cli, "--input", p, "--eps", 1, "--min-pts", 0)
    assert r.returncode == 2 and "min_pts must be >= 1" in r.stderr
    r = run(cli, "--input", p, "--eps", "x", "--min-pts", 1)
    assert r.returncode == 2 and "not a number" in r.stderr
    r = run(cli, "--input", p, "--eps", 1, "--min-pts", 1, "--dist", "l7")
    assert r.returncode == 2 and "unknown distance 'l7'" in r.stderr
    r = run(cli, "--input", p, "--eps", 1, "--min-pts", 1, "--bogus", 3)
    assert r.returncode == 2 and "unknown flag --bogus" in r.stderr


def test_io_errors_exit_3(cli, tmp_path):
    r = run(cli, "--input", tmp_path / "missing.sngd", "--eps", 1, "--min-pts", 1)
    assert r.returncode == 3 and "cannot open" in r.stderr
    bad = tmp_path / "bad.sngd"
    bad.write_bytes(b"SNGD\x02" + b"\0" * 16)
    r = run(cli, "--input", bad, "--eps", 1, "--min-pts", 1)
    assert r.returncode == 3 and "unsupported SNGD version 2" in r.stderr
    csv = tmp_path / "pts.csv"
    csv.write_text("0,1\n2,3\n")
    r = run(cli, "--input", csv, "--eps", 1, "--min-pts", 1)
    assert r.returncode == 3 and "not an SNGD dataset" in r.stderr


def test_no_gpu_fails_loudly(cli, tmp_path):
    if sng.device_count() > 0:
        pytest.skip("a GPU is present")
    r = run(cli, "--input", _line4(tmp_path), "--eps", 1, "--min-pts", 1)
    assert r.returncode == 1 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_spec_example(cli, tmp_path):
    p = _line4(tmp_path)
    out = tmp_path / "labels.txt"
    r = run(cli, "--input", p, "--eps", 1, "--min-pts", 1, "--rate", 1, "--output", out)
    assert r.returncode == 0, r.stderr
    assert out.read_text() == "0\n0\n1\n1\n"
    m = dict(kv.split("=") for kv in r.stdout.split())
    assert (m["n"], m["k"], m["noise"], m["edges"], m["evals"]) == ("4", "2", "0", "2", "12")
    r = run(cli, "--input", p, "--eps", 1, "--min-pts", 1, "--exact", "--output", out)
    assert r.returncode == 0 and "evals=6" in r.stdout and out.read_text() == "0\n0\n1\n1\n"
    # k = 0 is success
    r = run(cli, "--input", p, "--eps", 0.1, "--min-pts", 1, "--output", out)
    assert r.returncode == 0 and re.search(r"\bk=0\b", r.stdout)
    assert out.read_text() == "-1\n" * 4


@pytest.mark.gpu
def test_synthetic_against_oracle(cli, tmp_path, oracle):
    from paper_2006_06743_b200 import synthetic
    w = synthetic.CONFIGS[1]
    pts = synthetic.generate(1, n=5000)
    p = tmp_path / "cfg1.sngd"
    sio.save_binary(sng.Dataset(pts), str(p))
    out = tmp_path / "cfg1.labels"
    r = run(cli, "--input", p, "--eps", w.eps, "--min-pts", w.min_pts, "--rate", w.rate,
            "--seed", w.seed, "--output", out)
    assert r.returncode == 0, r.stderr
    labels, _, info, _ = oracle.sng_dbscan(pts, w.eps, w.min_pts, w.rate, w.seed)
    np.testing.assert_array_equal(sio.load_labels(str(out)), labels)
    m = dict(kv.split("=") for kv in r.stdout.split())
    assert int(m["edges"]) == info["edges"] and int(m["evals"]) == info["distance_evals"]
