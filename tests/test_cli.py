"""CLI front end (reference cli.py:149-261): argument parsing on CPU, the
gen -> svd / svd-naive / rpca / bench round trips on the GPU."""

import csv
import io
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_parse_helpers_match_reference_semantics():
    from paper_1706_07191_b200 import cli
    assert cli.parse_bytes("128MiB") == 128 << 20
    assert cli.parse_bytes("1g") == 10 ** 9
    assert cli.parse_bytes("4096") == 4096
    assert cli.parse_ratio("1024:32:1") == (1024, 32, 1)
    # synth.shape_from_ratio (synth.py:38-47): scale rounded down
    m, n, k = cli.shape_from_ratio((1024, 32, 1), 64 << 20, 8)
    assert (m, n, k) == (1024 * 16, 32 * 16, 16) and m * n * 8 <= 64 << 20
    ap = cli.build_parser()
    a = ap.parse_args(["svd", "--input", "x.oocm", "--rank", "5", "--partitions", "3",
                       "--memory-budget", "1MiB"])
    assert (a.rank, a.partitions, a.memory_budget, a.power) == (5, 3, 1 << 20, 1)


def test_errors_map_to_exit_code_1(tmp_path, capsys):
    """cli.py:280-282: ValueError / OSError -> exit status 1."""
    from paper_1706_07191_b200 import cli
    rc = cli.main(["svd", "--input", str(tmp_path / "missing.oocm"), "--rank", "3"])
    assert rc == 1
    assert "blocksvd-b200:" in capsys.readouterr().err


@pytest.mark.gpu
def test_gen_svd_and_naive_round_trip(tmp_path, capsys):
    from paper_1706_07191_b200 import cli
    path = str(tmp_path / "a.oocm")
    assert cli.main(["gen", "--m", "3000", "--n", "700", "--k", "12", "--out", path]) == 0
    capsys.readouterr()
    for cmd in ("svd", "svd-naive"):
        rc = cli.main([cmd, "--input", path, "--rank", "12", "--power", "1",
                       "--memory-budget", "4MiB", "--report", str(tmp_path / "r.json")])
        assert rc == 0
        rep = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
        # exact rank-12 matrix: the rank-12 factors reproduce it
        assert rep["relative_frobenius_error"] < 1e-10
        assert rep["full_passes"] == (2.0 if cmd == "svd" else 4.0)
        assert rep["a_stream_gbs"] > 0 and rep["boundary_words_read"] > 0
        with open(tmp_path / "r.json") as f:
            assert json.load(f)["m"] == 3000


@pytest.mark.gpu
def test_rpca_and_bench(tmp_path, capsys):
    from oracle import ref_cpu
    from paper_1706_07191_b200 import MatrixStore, cli
    a = ref_cpu.lowrank_plus_noise(300, 120, 3, 0.0, seed=2)
    a[np.random.default_rng(0).random(a.shape) < 0.02] += 5.0
    path = str(tmp_path / "m.oocm")
    MatrixStore.from_array(path, a, overwrite=True).close()
    lo = str(tmp_path / "L.oocm")
    rc = cli.main(["rpca", "--input", path, "--rank", "5", "--output-lowrank", lo])
    assert rc == 0
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert out["converged"] and out["iterations"] >= 1
    assert MatrixStore(lo).read_full().shape == a.shape
    rc = cli.main(["bench", "--ratios", "64:16:1", "--sizes", "2MiB", "--memory-budget",
                   "1MiB", "--workdir", str(tmp_path)])
    assert rc == 0
    rows = list(csv.DictReader(io.StringIO(capsys.readouterr().out)))
    assert [r["variant"] for r in rows] == ["proposed", "naive"]
    assert all(float(r["error"]) < 1e-8 for r in rows)
