"""CLI and vector files (reference cli.py / vecio.py; SPEC.md cli_io module).

CPU tests: vector file round trips and error handling, argument validation
and exit codes, `params` output (host planner only).  GPU tests: `transform`
and `bench` end to end through the CUDA path.
"""

import math
import struct

import numpy as np
import pytest

import paper_1501_01652_b200 as fh
from paper_1501_01652_b200 import cli, vecio


# --------------------------------------------------------------- vector files
@pytest.mark.parametrize("fmt", ["text", "binary"])
def test_vector_round_trip_bit_exact(tmp_path, fmt):
    rng = np.random.default_rng(7)
    v = np.concatenate([rng.standard_normal(257) * 10.0 ** rng.integers(-300, 300, 257),
                        [0.0, -0.0, 1e-310, np.pi, -1.0 / 3.0, 2.0 ** -1074, 1.7976931348623157e308]])
    p = tmp_path / ("v." + fmt)
    fh.write_vector(str(p), v, fmt)
    w = fh.read_vector(str(p), fmt)
    assert w.dtype == np.float64 and w.shape == v.shape
    assert np.array_equal(w.view(np.uint64), v.view(np.uint64))


def test_binary_layout(tmp_path):
    p = tmp_path / "v.bin"
    vecio.write_vector(str(p), [1.5, -2.0], "binary")
    blob = p.read_bytes()
    assert blob[:4] == b"FHK1"
    assert struct.unpack("<Q", blob[4:12]) == (2,)
    assert struct.unpack("<2d", blob[12:]) == (1.5, -2.0)


def test_text_comments_and_blank_lines(tmp_path):
    p = tmp_path / "v.txt"
    p.write_text("# header\n\n1.25  # trailing\n   \n-3e2\n#only\n7\n")
    assert list(vecio.read_vector(str(p))) == [1.25, -300.0, 7.0]


def test_text_written_with_17_digits(tmp_path):
    p = tmp_path / "v.txt"
    vecio.write_vector(str(p), [0.1], "text")
    assert p.read_text() == "0.10000000000000001\n"


@pytest.mark.parametrize("blob,msg", [
    (b"FHK", "truncated"),
    (b"XXXX" + struct.pack("<Q", 0), "bad magic"),
    (b"FHK1" + struct.pack("<Q", 2) + struct.pack("<d", 1.0), "expected"),
    (b"FHK1" + struct.pack("<Q", 0) + b"\x00", "expected"),
])
def test_binary_malformed(tmp_path, blob, msg):
    p = tmp_path / "bad.bin"
    p.write_bytes(blob)
    with pytest.raises(vecio.VectorFileError, match=msg):
        vecio.read_vector(str(p), "binary")


def test_text_malformed(tmp_path):
    p = tmp_path / "bad.txt"
    p.write_text("1.0\n2.0\nabc\n")
    with pytest.raises(vecio.VectorFileError, match=r":3: not a number"):
        vecio.read_vector(str(p))
    q = tmp_path / "bin.txt"
    q.write_bytes(b"\xff\xfe\x00\x01")
    with pytest.raises(vecio.VectorFileError):
        vecio.read_vector(str(q))
    with pytest.raises(vecio.VectorFileError):
        vecio.read_vector(str(tmp_path / "missing.txt"))


def test_vector_argument_errors(tmp_path):
    with pytest.raises(ValueError):
        vecio.write_vector(str(tmp_path / "a"), np.zeros((2, 2)))
    with pytest.raises(ValueError):
        vecio.write_vector(str(tmp_path / "a"), [1.0], "csv")
    with pytest.raises(ValueError):
        vecio.read_vector(str(tmp_path / "a"), "csv")


# ------------------------------------------------------------ CLI, host side
def _params(capsys, *argv):
    assert cli.main(["params", *argv]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    return dict(line.split("=", 1) for line in out)


def test_params_schlomilch_table4(capsys):
    kv = _params(capsys, "schlomilch", "--n", "10000", "--eps", "1e-15")
    assert kv["M"] == "10"                                        # SPEC cmd_params example
    kv = _params(capsys, "schlomilch", "--nu", "4", "--gamma", "4", "--n", str(2 ** 20), "--eps", "1e-15")
    assert kv["M"] == "10" and kv["P"] == "3" and abs(float(kv["s"]) - 18.5378) < 1e-3


def test_params_fourier_bessel_and_dht(capsys):
    kv = _params(capsys, "fourier-bessel", "--n", "4096", "--eps", "1e-15")
    assert kv["K"] == "6" and kv["T"] == "3" and kv["n_split"] == "22"
    kv = _params(capsys, "dht", "--n", str(2 ** 16), "--eps", "1e-15")
    assert kv["row_split"] == "22"                                # floor(1.01 * 22.76)
    # the engine dht() really uses (M=11, s=25.540, P=3)
    assert kv["M"] == "11" and kv["P"] == "3" and abs(float(kv["s"]) - 25.540) < 1e-3


@pytest.mark.parametrize("argv", [
    ["params", "schlomilch", "--n", "100", "--eps", "1.5"],
    ["params", "schlomilch", "--n", "100", "--eps", "1e-17"],
    ["params", "schlomilch", "--n", "0"],
    ["params", "dht", "--n", "10", "--nu", "-1"],
    ["params", "schlomilch"],                                     # --n required
    ["transform", "dht", "a", "b", "--eps", "2"],                 # SPEC: dht eps out of range -> 1
    ["transform", "dht", "a", "b", "--nu", "1"],
    ["transform", "fourier-bessel", "a", "b", "--gamma", "0.5"],
    ["transform", "fourier-bessel", "a", "b", "--method", "single"],
    ["transform", "schlomilch", "a", "b", "--threads", "0"],
    ["bench", "schlomilch", "--sizes", ""],                       # SPEC: empty N-list -> 1
    ["bench", "schlomilch", "--sizes", "4,x"],
    ["bench", "schlomilch", "--sizes", "0"],
    ["bench", "schlomilch", "--sizes", "8", "--self-inverse"],
    ["frobnicate"],
])
def test_usage_errors_exit_1(argv, capsys):
    assert cli.main(argv) == cli.EXIT_USAGE
    assert capsys.readouterr().err.startswith("fasthankel: ")


def test_unreadable_input_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.txt"
    bad.write_text("1.0\nnope\n")
    assert cli.main(["transform", "schlomilch", str(bad), str(tmp_path / "o")]) == cli.EXIT_INPUT
    assert cli.main(["transform", "schlomilch", str(tmp_path / "none"), str(tmp_path / "o")]) == cli.EXIT_INPUT
    empty = tmp_path / "empty.txt"
    empty.write_text("# nothing\n")
    assert cli.main(["transform", "schlomilch", str(empty), str(tmp_path / "o")]) == cli.EXIT_INPUT


# ------------------------------------------------------------- CLI on the GPU
@pytest.mark.gpu
def test_transform_single_value_is_j0_pi(tmp_path, cuda_dev):
    src, dst = tmp_path / "c.txt", tmp_path / "f.txt"
    fh.write_vector(str(src), [1.0])
    assert cli.main(["transform", "schlomilch", str(src), str(dst)]) == 0
    from oracle import fht_oracle as ora
    f = fh.read_vector(str(dst))
    assert f.shape == (1,)
    assert abs(f[0] - ora.besselj(0, np.array([math.pi]))[0]) < 1e-15


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n", [("schlomilch", 300), ("fourier-bessel", 900), ("dht", 200)])
@pytest.mark.parametrize("fmt", ["text", "binary"])
def test_transform_fast_matches_direct(tmp_path, cuda_dev, kind, n, fmt):
    rng = np.random.default_rng([3, n])
    c = rng.standard_normal(n)
    src = tmp_path / "c"
    fh.write_vector(str(src), c, fmt)
    outs = {}
    for method in ("direct", "fast"):
        dst = tmp_path / method
        assert cli.main(["transform", kind, str(src), str(dst), "--method", method, "--format", fmt]) == 0
        outs[method] = fh.read_vector(str(dst), fmt)
    eps = 1e-15
    assert np.max(np.abs(outs["fast"] - outs["direct"])) <= 10 * eps * np.abs(c).sum()


@pytest.mark.gpu
def test_transform_matches_library_call(tmp_path, cuda_dev):
    c = np.random.default_rng(11).standard_normal(700)
    src, dst = tmp_path / "c.bin", tmp_path / "f.bin"
    fh.write_vector(str(src), c, "binary")
    assert cli.main(["transform", "schlomilch", str(src), str(dst), "--nu", "2", "--gamma", "0.5",
                     "--eps", "1e-8", "--format", "binary"]) == 0
    ref = fh.schlomilch_fast(fh.select_params(2, 700, 1e-8, 0.5), c)
    assert np.array_equal(fh.read_vector(str(dst), "binary"), ref)   # deterministic


@pytest.mark.gpu
def test_bench_csv(capsys, cuda_dev):
    assert cli.main(["bench", "schlomilch", "--sizes", "128,512", "--eps", "1e-15"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "N,method,seconds,max_abs_error_vs_direct"
    body = [r.split(",") for r in rows[1:]]
    assert [(r[0], r[1]) for r in body] == [("128", "direct"), ("128", "single"), ("128", "fast"),
                                            ("512", "direct"), ("512", "single"), ("512", "fast")]
    for n, method, sec, err in body:
        c = np.random.default_rng([0, int(n)]).standard_normal(int(n))
        assert float(sec) >= 0.0
        assert float(err) <= 10 * 1e-15 * np.abs(c).sum()
    assert cli.main(["bench", "dht", "--sizes", "64", "--self-inverse", "--direct-cap", "0"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[1].startswith("64,fast,") and rows[1].endswith(",")   # direct skipped: no error column
    assert rows[2].startswith("64,self-inverse,")


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n", [("schlomilch", 300), ("schlomilch", 40), ("dht", 200)])
def test_transform_non_finite_output_exit_3(tmp_path, cuda_dev, capsys, kind, n):
    """Reference cli.py:128-130: a non-finite output value is exit code 3 and
    no output file.  Here the flag is raised on the device by the reductions
    that write the output (fhtb_nonfinite_check -> FHTB_ENONFINITE)."""
    c = np.random.default_rng([5, n]).standard_normal(n)
    c[n // 2] = np.inf
    src, dst = tmp_path / "c.bin", tmp_path / "f.bin"
    fh.write_vector(str(src), c, "binary")
    assert cli.main(["transform", kind, str(src), str(dst), "--format", "binary"]) == 3
    assert "non-finite" in capsys.readouterr().err
    assert not dst.exists()
    # the flag is cleared by the check: a clean vector afterwards is exit 0
    c[n // 2] = 1.0
    fh.write_vector(str(src), c, "binary")
    assert cli.main(["transform", kind, str(src), str(dst), "--format", "binary"]) == 0
