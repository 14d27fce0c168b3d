"""The GPU-path CLI (tools/cli/wavelcs_b200_main.cpp)
and the input path behind it (load_sequence / parse_fasta semantics of the
reference's io.cpp:46-101), mirroring proj/tests/test_cli.cpp and
test_io.cpp.  `gen` and argument errors need no GPU; compute/bench do."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1306_4627_b200", "_lib", "wavelcs_b200")


def run(*args):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout + p.stderr


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(CLI):
        pytest.skip("CLI not built (make all)")


def test_gen_matches_reference_generator(tmp_path, restatement):
    out = tmp_path / "g.txt"
    rc, _ = run("gen", "--length", "1000", "--alphabet", "ACGT", "--seed", "42", "--out", str(out))
    assert rc == 0
    assert out.read_bytes() == restatement.generate_random(1000, b"ACGT", 42)


def test_argument_errors():
    rc, text = run("nonsense")
    assert rc == 1 and "error:" in text
    rc, text = run("gen", "--length", "5")
    assert rc == 1 and "error:" in text
    rc, text = run("compute", "--parent")
    assert rc == 1 and "error:" in text


@pytest.mark.gpu
def test_compute_identical_inputs(tmp_path):
    # test_cli.cpp:71-80
    (tmp_path / "p.txt").write_text("ATGC\n")
    (tmp_path / "c.txt").write_text("ATGC\n")
    rc, text = run("compute", "--parent", str(tmp_path / "p.txt"), "--child", str(tmp_path / "c.txt"))
    assert rc == 0 and "LCS length:  4" in text and "100.00%" in text


@pytest.mark.gpu
def test_compute_traceback_and_worker_flags(tmp_path):
    # test_cli.cpp:82-112
    (tmp_path / "p.txt").write_text("ABCBDAB")
    (tmp_path / "c.txt").write_text("BDCABA")
    args = ["--traceback", "--parent", str(tmp_path / "p.txt"), "--child", str(tmp_path / "c.txt")]
    rc, text = run("compute", *args)
    assert rc == 0 and "LCS length:  4" in text and "LCS:         BDAB" in text
    rc2, text2 = run("compute", "--workers", "7", "--block-size", "3", *args)
    pick = lambda t, pre: next(l for l in t.splitlines() if l.startswith(pre))
    for pre in ("LCS length", "Similarity", "LCS:"):
        assert pick(text, pre) == pick(text2, pre)


@pytest.mark.gpu
def test_compute_fasta_and_whitespace(tmp_path):
    # FASTA: first record only, upper-cased, whitespace dropped; plain:
    # every ASCII space stripped (io.cpp:46-101)
    (tmp_path / "p.fa").write_text(">one\nabc b\nDAB\n>two\nTTTT\n")
    (tmp_path / "c.txt").write_text("BD CA\n\tBA\r\n")
    rc, text = run("compute", "--traceback", "--parent", str(tmp_path / "p.fa"),
                   "--child", str(tmp_path / "c.txt"))
    assert rc == 0 and "LCS:         BDAB" in text
    (tmp_path / "bad.fa").write_text("ACGT\n>late\n")
    rc, text = run("compute", "--parent", str(tmp_path / "bad.fa"), "--child", str(tmp_path / "c.txt"))
    assert rc == 1 and "malformed FASTA" in text
    rc, text = run("compute", "--validate-dna", "--parent", str(tmp_path / "p.fa"),
                   "--child", str(tmp_path / "c.txt"))
    assert rc == 1 and "outside the {A, C, G, T} alphabet" in text
    rc, text = run("compute", "--parent", str(tmp_path / "missing.txt"), "--child", str(tmp_path / "c.txt"))
    assert rc == 1 and "cannot open" in text


@pytest.mark.gpu
def test_bench_csv_gcups(tmp_path):
    """--gcups: the device throughput schema (GCUPS, fraction of the int roofline)."""
    out = tmp_path / "b.csv"
    rc, text = run("bench", "--gcups", "--sizes", "1000x1000,10000x10000", "--repetitions", "2",
                   "--out", str(out))
    assert rc == 0
    rows = [l for l in out.read_text().splitlines() if l and not l.startswith("#")]
    assert rows[0] == "M,N,repetitions,device_s,gcups,roofline_frac,lcs_length"
    assert rows[2].split(",")[-1] == "6538"  # SURVEY 8(c) checkpoint, seed 1


@pytest.mark.gpu
def test_bench_csv_reference_schema(tmp_path):
    """Default: the reference's bench (proj/src/bench.cpp:71-162) -- serial and
    parallel fills with the equivalence gate, the 8-column CSV."""
    out = tmp_path / "r.csv"
    rc, text = run("bench", "--sizes", "10000x1000,100x10", "--workers", "1,4", "--repetitions", "1",
                   "--seed", "1", "--out", str(out))
    assert rc == 0, text
    lines = out.read_text().splitlines()
    assert lines[0] == "# wavelcs benchmark"
    rows = [l for l in lines if l and not l.startswith("#")]
    assert rows[0] == "M,N,workers,block_size,serial_s,parallel_s,speedup,lcs_length"
    assert len(rows) == 5
    assert rows[1].split(",")[-1] == rows[3].split(",")[-1]  # workers do not change the length
