"""OLS1 sample files and the CLI (reference io.py / cli.py).

CPU: byte-level compatibility with files written by the reference's own
writer (tests/golden/io), header validation, argument parsing and I/O error
exit codes.  GPU (-m gpu): the subcommands end to end.
"""

import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

from paper_1910_01972_b200 import Precision
from paper_1910_01972_b200.cli import CSV_HEADER, build_parser, main
from paper_1910_01972_b200.io import read_samples, write_samples

IO = os.path.join(GOLDEN, "io")
NAMES = ["real_single", "real_double", "complex_single", "complex_double"]


@pytest.mark.parametrize("name", NAMES)
def test_reads_reference_files_and_writes_identical_bytes(tmp_path, name):
    want = np.load(os.path.join(IO, "arrays.npz"))[name]
    kind = "complex" if "complex" in name else "real"
    prec = Precision.single if "single" in name else Precision.double
    for ext in (".bin", ".txt"):
        ref_file = os.path.join(IO, name + ext)
        got, k, p = read_samples(ref_file, prec)
        assert k == kind and p is prec and got.dtype == want.dtype
        assert np.array_equal(got, want)
        mine = tmp_path / (name + ext)
        write_samples(mine, want)
        assert mine.read_bytes() == open(ref_file, "rb").read()


def test_header_validation(tmp_path):
    good = (tmp_path / "g.bin")
    write_samples(good, np.arange(4, dtype=np.float32))
    raw = good.read_bytes()
    (tmp_path / "t.bin").write_bytes(raw[:10])
    with pytest.raises(ValueError, match="truncated"):
        read_samples(tmp_path / "t.bin")
    (tmp_path / "k.bin").write_bytes(raw[:4] + bytes([7]) + raw[5:])
    with pytest.raises(ValueError, match="bad header"):
        read_samples(tmp_path / "k.bin")
    (tmp_path / "c.bin").write_bytes(raw[:8] + struct.pack("<Q", 5) + raw[16:])
    with pytest.raises(ValueError, match="expected 5 samples"):
        read_samples(tmp_path / "c.bin")
    (tmp_path / "w.txt").write_text("1 2\n3\n")
    with pytest.raises(ValueError, match="columns"):
        read_samples(tmp_path / "w.txt")
    (tmp_path / "e.txt").write_text("\n")
    with pytest.raises(ValueError, match="no samples"):
        read_samples(tmp_path / "e.txt")


def test_parser_matches_reference_options():
    p = build_parser()
    a = p.parse_args(["convolve", "x.bin", "h.bin", "-o", "y.bin",
                      "--filter-len", "5", "--postproc", "derivative"])
    assert (a.command, a.filter_len, a.postproc, a.fft_len, a.variant) == (
        "convolve", 5, "derivative", "auto", "fused")
    a = p.parse_args(["verify", "--ns", "10,20", "--filters", "1,3",
                      "--centred"])
    assert a.ns == [10, 20] and a.filters == [1, 3] and a.centred
    a = p.parse_args(["tune", "--filter-len", "65,257"])
    assert a.filter_len == [65, 257] and a.mode == "r2r"
    assert CSV_HEADER.split(",")[-2:] == ["wall_time_s", "elements_per_s"]


def test_missing_file_exit_code(tmp_path, capsys):
    rc = main(["convolve", str(tmp_path / "nope.bin"), str(tmp_path / "h.bin"),
               "-o", str(tmp_path / "y.bin")])
    assert rc == 2
    assert "no such file" in capsys.readouterr().err


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1910_01972_b200.cli",
                           *args], cwd=ROOT, capture_output=True, text=True,
                          timeout=600)


@pytest.mark.gpu
def test_cli_convolve_matches_api(tmp_path):
    import paper_1910_01972_b200 as oc
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(5000) + 1j * rng.standard_normal(5000)).astype(
        np.complex64)
    taps = (rng.standard_normal((2, 33)) + 1j * rng.standard_normal((2, 33))
            ).astype(np.complex64)
    write_samples(tmp_path / "x.bin", x)
    write_samples(tmp_path / "h.bin", taps.reshape(-1))
    r = _cli("convolve", str(tmp_path / "x.bin"), str(tmp_path / "h.bin"),
             "-o", str(tmp_path / "y.bin"), "--filters", "2", "--fft-len", "256",
             "--origin", "3")
    assert r.returncode == 0, r.stderr
    P = Precision.single
    want = oc.convolve(oc.make_signal(x, "complex", P),
                       oc.make_filterset(taps, 3, P),
                       oc.plan(5000, 33, "c2c", 3, 256)).cpu().numpy()
    for f in range(2):
        got, kind, _ = read_samples(tmp_path / f"y.f{f}.bin")
        assert kind == "complex" and np.array_equal(got, want[f])


@pytest.mark.gpu
def test_cli_verify_bench_tune(tmp_path):
    r = _cli("verify", "--ns", "1000,20000", "--filter-len", "3,64,257",
             "--filters", "1,3")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cases passed" in r.stdout and "FAIL" not in r.stdout
    r = _cli("verify", "--ns", "1000", "--filter-len", "64", "--filters", "1",
             "--corrupt")
    assert r.returncode == 1
    cfg = tmp_path / "sweep.json"
    cfg.write_text('{"ns": [100000], "m": [65], "nfil": [2], "modes": '
                   '["c2c", "r2r"], "repeats": 2, "warmup": 1}')
    csv = tmp_path / "out.csv"
    r = _cli("bench", str(cfg), "--csv", str(csv))
    assert r.returncode == 0, r.stderr
    lines = csv.read_text().splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == 5     # 2 modes x 2 variants
    assert all(float(ln.split(",")[-1]) > 0 for ln in lines[1:])
    r = _cli("tune", "--filter-len", "65", "--probe-len", "65536",
             "--candidates", "128,256,1024")
    assert r.returncode == 0, r.stderr
    assert "best_n=" in r.stdout
