"""CLI and text formats against the reference's own CLI
outputs (tests/golden/cli, made by tests/golden/make_golden_cli.py)."""

import csv
from pathlib import Path

import numpy as np
import pytest

from oracle import covoracle as co
from paper_1303_2285_b200.cli import main
from paper_1303_2285_b200.io import (
    format_entry,
    parse_entry,
    read_covariance,
    read_input_matrix,
    write_covariance,
    write_input_matrix,
)

GOLD = Path(__file__).resolve().parent / "golden" / "cli"


def run(*argv):
    return main([str(a) for a in argv])


def test_gen_is_byte_identical_to_reference(tmp_path):
    out = tmp_path / "g.txt"
    assert run("--cmd", "gen", "--n", 9, "--m", 7, "--seed", 7, "--out", out) == 0
    assert out.read_bytes() == (GOLD / "gen_9x7_s7.txt").read_bytes()


def test_count_matches_reference(tmp_path):
    out = tmp_path / "c.csv"
    assert run("--cmd", "count", "--n", 32, "--m", 32, "--p", 13, "--q", 13, "--out", out) == 0
    assert out.read_text() == (GOLD / "count_32_13.csv").read_text().replace("\r\n", "\n") or \
        list(csv.reader(out.open())) == list(csv.reader((GOLD / "count_32_13.csv").open()))


def test_reference_estimate_file_reads_back_and_matches_oracle():
    a = read_input_matrix(GOLD / "gen_9x7_s7.txt")
    dense = read_covariance(GOLD / "estimate_9x7_p3q2.txt")
    assert np.array_equal(dense, dense.conj().T)
    ref = co.dense_from_packed(co.estimate_packed(a, 3, 2), 6)
    assert co.rel_frobenius(dense, ref) <= 1e-15


def test_entry_format_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    vals = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    vals[0] = 0.0
    vals[1] = -0.0 + 1e-300j
    for z in vals:
        assert parse_entry(format_entry(complex(z))) == complex(z)
    a = vals.reshape(5, 10)
    write_input_matrix(a, tmp_path / "a.txt")
    assert np.array_equal(read_input_matrix(tmp_path / "a.txt"), a)
    g = a @ a.conj().T
    h = co.dense_from_packed(g[np.triu_indices(5)], 5)  # exactly Hermitian
    write_covariance(h, tmp_path / "h.txt")
    assert np.array_equal(read_covariance(tmp_path / "h.txt"), h)
    with pytest.raises(ValueError):
        parse_entry("1.0+2.0")


def test_usage_errors(tmp_path, capsys):
    assert run("--cmd", "gen", "--n", 4) == 2
    err = capsys.readouterr().err
    assert "--m" in err and "--out" in err
    with pytest.raises(SystemExit) as exc:
        run("--cmd", "gen", "--n", 0, "--m", 4, "--out", tmp_path / "x.txt")
    assert exc.value.code == 2
    assert run("--cmd", "count", "--n", 4, "--m", 4, "--p", 5, "--q", 1) == 2
    assert run("--cmd", "estimate", "--in", tmp_path / "missing.txt", "--p", 2, "--q", 2,
               "--out", tmp_path / "c.txt") == 2


@pytest.mark.gpu
def test_gpu_estimate_raw_matches_reference_file(cuda, tmp_path):
    out = tmp_path / "r.txt"
    assert run("--cmd", "estimate", "--in", GOLD / "gen_9x7_s7.txt", "--p", 3, "--q", 2,
               "--raw", "--out", out) == 0
    got = read_covariance(out)
    ref = read_covariance(GOLD / "estimate_9x7_p3q2.txt")
    assert co.rel_frobenius(got, ref) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--complex64"]])
def test_gpu_verify_and_bench(cuda, tmp_path, extra):
    out = tmp_path / "v.csv"
    assert run("--cmd", "verify", "--n", 40, "--m", 33, "--p", 7, "--q", 5, "--threads", 3,
               "--out", out, *extra) == 0
    rows = list(csv.reader(out.open()))
    assert rows[0] == ["comparison", "max_rel_diff", "pass"]
    assert all(r[2] == "pass" for r in rows[1:])
    trace = tmp_path / "t.csv"
    bench = tmp_path / "b.csv"
    assert run("--cmd", "bench", "--n", 64, "--m", 64, "--p", 8, "--q", 8, "--repeats", 2,
               "--out", bench, "--trace-out", trace, *extra) == 0
    b = list(csv.reader(bench.open()))
    assert [r[0] for r in b[1:]] == ["naive", "seq", "seq-opt", "par"]
    t = list(csv.reader(trace.open()))
    assert t[0] == ["task_id", "dr", "dc", "cost"] and len(t) == 1 + 8 * 8 + 7 * 7
    assert all(float(r[3]) > 0 for r in t[1:])
