"""`build/pixelseg_gpu` (tools/pixelseg_gpu.cpp): the reference CLI's process / bench / sizes /
flops subcommands (proj/tools/pixelseg.cpp) on the B200 path.

Fixtures (tests/golden/cli/, made by `make_golden.py cli` from the reference itself): a
reduced-channel sk.net spec file, PXSG weights written by the reference's save_weights, a 300x260
scan written by the reference's write_pgm (and the same pixels as PNG), and the output files the
reference's process<float> gives at the default tile (labels PGM, 8-bit probability maps)."""
import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, config_text

BIN = os.path.join(ROOT, "build", "pixelseg_gpu")
CLI = os.path.join(GOLDEN, "cli")
needs_bin = pytest.mark.skipif(not os.path.exists(BIN),
                               reason="build/pixelseg_gpu not built (needs /root/reference at build time)")


def run(*args, timeout=600):
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=timeout)


def read_pgm(path):
    """Binary P5 maxval-255 reader (the format write_pgm emits, image_io.hpp:83-93)."""
    data = open(path, "rb").read()
    toks, pos = [], 0
    while len(toks) < 4:
        while data[pos:pos + 1].isspace():
            pos += 1
        if data[pos:pos + 1] == b"#":
            pos = data.index(b"\n", pos) + 1
            continue
        end = pos
        while not data[end:end + 1].isspace():
            end += 1
        toks.append(data[pos:end])
        pos = end
    assert toks[0] == b"P5" and toks[3] == b"255"
    w, h = int(toks[1]), int(toks[2])
    return np.frombuffer(data[pos + 1:pos + 1 + w * h], np.uint8).reshape(h, w)


# ---- host-only subcommands (no GPU) ---------------------------------------------------------

@needs_bin
def test_cli_flops_matches_reference_table(tmp_path):
    net = tmp_path / "sk.net"
    net.write_text(config_text("sk"))
    r = run("flops", "--net", str(net))
    assert r.returncode == 0, r.stderr
    rows = dict(line.split("\t") for line in r.stdout.splitlines() if not line.startswith("#"))
    # flop_estimate(sk.net, 229) (convert.hpp:308-322); total = SURVEY.md §8 a18
    assert rows["ip1"] == "644228317184"
    assert rows["total"] == "694596973808"


@needs_bin
def test_cli_sizes_output_extent(tmp_path):
    net = tmp_path / "sk.net"
    net.write_text(config_text("sk"))
    r = run("sizes", "--net", str(net), "--w0", "1125")
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().splitlines()[-1] == "# output extent: 1024"


@needs_bin
def test_cli_exit_codes(tmp_path):
    assert run().returncode == 1                                      # no subcommand
    assert run("frobnicate").returncode == 1                          # usage
    assert run("flops").returncode == 1                               # --net required
    r = run("flops", "--net", str(tmp_path / "missing.net"))
    assert r.returncode == 3 and "cannot open" in r.stderr           # IoError
    bad = tmp_path / "bad.net"
    bad.write_text("input w=10 f=1\nlayer c conv_sk k=3 fout=0 in=data out=c\n")
    assert run("flops", "--net", str(bad)).returncode == 2            # SpecError
    assert run("bench", "--net", str(bad), "--backward").returncode == 2  # SpecError first
    assert run("process", "--net", str(bad), "--weights", "w", "--in", "i", "--out", "o",
               "--gpus", "0").returncode == 1                       # usage


# ---- process / bench on the GPU -------------------------------------------------------------

@pytest.mark.gpu
@needs_bin
@pytest.mark.parametrize("image", ["scan.pgm", "scan.png"])
def test_cli_process_matches_reference_files(tmp_path, image):
    src = tmp_path / image
    shutil.copy(os.path.join(CLI, image), src)
    out = tmp_path / "out"
    r = run("process", "--net", os.path.join(CLI, "sk_small.net"), "--weights",
            os.path.join(CLI, "sk_small.pxsg"), "--in", str(src), "--out", str(out), "--prob")
    assert r.returncode == 0, r.stderr
    assert r.stdout.splitlines() == [f"wrote\t{out}/scan_labels.pgm", f"wrote\t{out}/scan_prob0.pgm",
                                     f"wrote\t{out}/scan_prob1.pgm"]
    for name in ("labels", "prob0", "prob1"):
        got = open(out / f"scan_{name}.pgm", "rb").read()
        want = open(os.path.join(CLI, f"expect_scan_{name}.pgm"), "rb").read()
        assert got == want, f"{name}: output file differs from the reference's"


@pytest.mark.gpu
@needs_bin
@pytest.mark.parametrize("tile", [64, 37, 260])
def test_cli_process_any_tile_same_labels(tmp_path, tile):
    """The labelling does not depend on the tile (pipeline.hpp:662-672; test_pipeline.cpp:535-588)."""
    out = tmp_path / "out"
    r = run("process", "--net", os.path.join(CLI, "sk_small.net"), "--weights",
            os.path.join(CLI, "sk_small.pxsg"), "--in", os.path.join(CLI, "scan.pgm"), "--out",
            str(out), "--tile", str(tile))
    assert r.returncode == 0, r.stderr
    assert np.array_equal(read_pgm(out / "scan_labels.pgm"),
                          read_pgm(os.path.join(CLI, "expect_scan_labels.pgm")))


@pytest.mark.gpu
@needs_bin
def test_cli_process_weights_mismatch_is_spec_error(tmp_path):
    net = tmp_path / "sk.net"
    net.write_text(config_text("sk"))  # full-width sk.net vs reduced-width weights
    r = run("process", "--net", str(net), "--weights", os.path.join(CLI, "sk_small.pxsg"), "--in",
            os.path.join(CLI, "scan.pgm"), "--out", str(tmp_path / "o"))
    assert r.returncode in (2, 3), r.stderr
    assert r.stderr.startswith("error: ")


@pytest.mark.gpu
@needs_bin
def test_cli_bench_report(tmp_path):
    r = run("bench", "--net", os.path.join(CLI, "sk_small.net"), "--trials", "2",
            "--peak-gflops", "37000")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "# forward timing: input 229, output 128, 2 trials, seed 1"
    rows = {tuple(line.split("\t")[:2]): line.split("\t")[2] for line in lines[1:]}
    assert rows[("output", "extent")] == "128"
    assert float(rows[("throughput", "px_per_s")]) > 0
    assert ("ip1", "efficiency") in rows and ("total", "gflops") in rows


TIMING = {"seconds", "gflops", "efficiency", "px_per_s"}


def strip_timing(text):
    """The bench report without its timing columns (acceptance.cpp:1159-1166 compares the rest)."""
    return [ln for ln in text.splitlines() if not (len(ln.split("\t")) == 3 and ln.split("\t")[1] in TIMING)]


@pytest.mark.gpu
@needs_bin
def test_cli_determinism(tmp_path):
    """proj/tests/acceptance.cpp:1106-1178 on the GPU CLI: two identically seeded runs give
    byte-identical output files (process) and identical reports outside the timing columns
    (bench, forward and --backward)."""
    outs = []
    for i in range(2):
        out = tmp_path / f"o{i}"
        r = run("process", "--net", os.path.join(CLI, "sk_small.net"), "--weights",
                os.path.join(CLI, "sk_small.pxsg"), "--in", os.path.join(CLI, "scan.pgm"), "--out",
                str(out), "--prob")
        assert r.returncode == 0, r.stderr
        outs.append([open(out / f"scan_{n}.pgm", "rb").read() for n in ("labels", "prob0", "prob1")])
    assert outs[0] == outs[1]
    reports = []
    for i in range(2):
        r = run("bench", "--net", os.path.join(CLI, "sk_small.net"), "--w0", "130", "--trials", "2",
                "--seed", "5", "--backward")
        assert r.returncode == 0, r.stderr
        reports.append(r.stdout)
    assert strip_timing(reports[0]) == strip_timing(reports[1])
    rows = {tuple(ln.split("\t")[:2]): ln.split("\t")[2] for ln in reports[0].splitlines()[1:]}
    assert float(rows[("backward", "seconds")]) > 0


@pytest.mark.gpu
@needs_bin
@pytest.mark.parametrize("gpus", [2, 3])
def test_cli_process_gpus_same_files(tmp_path, gpus):
    """--gpus G: tile-row bands on G ranks (round-robin over the visible GPUs) give the
    reference's output files byte for byte."""
    out = tmp_path / "out"
    r = run("process", "--net", os.path.join(CLI, "sk_small.net"), "--weights",
            os.path.join(CLI, "sk_small.pxsg"), "--in", os.path.join(CLI, "scan.pgm"), "--out",
            str(out), "--prob", "--gpus", str(gpus))
    assert r.returncode == 0, r.stderr
    for name in ("labels", "prob0", "prob1"):
        assert open(out / f"scan_{name}.pgm", "rb").read() == \
            open(os.path.join(CLI, f"expect_scan_{name}.pgm"), "rb").read(), name
