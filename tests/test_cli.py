"""semd-cli: the reference CLI's `decompose` front-end (cli.cpp:93-134) over the B200 library.

CPU: the tool builds, its synth output and JSON number formatting equal the reference's bytes,
usage and input errors take the reference's exit codes and messages (no GPU needed: inputs are
parsed before the engine starts). GPU: every output file (per-mode CSV with %.17g, rescaled PGM,
sidecar JSON) is byte-identical to the reference pipeline's (tests/golden/cli.json, made by
tests/golden/make_golden_cli.py from the reference itself), EEMD and CEEMDAN included.
"""
import hashlib
import json
import os
import subprocess

import pytest

from tests.conftest import GOLDEN, ROOT
from tests.golden.make_golden_cli import make_inputs

CLI = os.path.join(ROOT, "paper_2106_15319_b200", "semd-cli")


@pytest.fixture(scope="module")
def cli():
    from paper_2106_15319_b200.csrc import build
    build.build()
    assert os.path.exists(CLI)
    return CLI


@pytest.fixture(scope="module")
def gold():
    return json.load(open(os.path.join(GOLDEN, "cli.json")))


def run(*args, cwd=None):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=600)


def sha_file(p):
    return hashlib.sha256(open(p, "rb").read()).hexdigest()


def test_synth_signals_bytes(cli, gold, tmp_path):
    r = run("synth", "signals", "--out", tmp_path)
    assert r.returncode == 0, r.stderr
    assert sha_file(tmp_path / "signals.csv") == gold["inputs"]["signals.csv"]
    make_inputs(str(tmp_path))
    assert sha_file(tmp_path / "texture.pgm") == gold["inputs"]["texture.pgm"]


def test_json_numbers_match_nlohmann(tmp_path):
    """io_detail::json_double (the sidecar's nstd) prints doubles exactly like nlohmann::json."""
    cases = json.load(open(os.path.join(GOLDEN, "cli.json")))["json_double"]
    src = tmp_path / "j.cpp"
    src.write_text('#include "semd/io.hpp"\n#include <cstdio>\n#include <cstdlib>\n'
                   'int main(int c, char** v) { for (int i = 1; i < c; ++i) '
                   'std::printf("%s\\n", semd::io_detail::json_double(std::strtod(v[i], nullptr)).c_str()); }\n')
    exe = tmp_path / "j"
    r = subprocess.run(["g++", "-std=c++20", "-I" + os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)] + [h for h, _ in cases], capture_output=True, text=True).stdout.split()
    assert out == [t for _, t in cases]


def test_usage_and_input_errors(cli, tmp_path):
    assert run("--help").returncode == 0
    assert run().returncode == 2
    assert run("frobnicate").returncode == 2
    assert run("decompose", "x.csv", "--bogus", "1").returncode == 2
    r = run("decompose", tmp_path / "missing.csv")
    assert r.returncode == 2 and "error: cannot open CSV file: " in r.stderr
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b\n1,2\n3,x\n")
    r = run("decompose", bad)
    assert r.returncode == 2 and r.stderr.strip() == f"error: cannot parse number 'x' at {bad}, line 3"
    bad.write_text("a,b\n1,2,3\n")
    assert run("decompose", bad).stderr.strip() == f"error: expected 2 fields, got 3 at {bad}, line 2"
    pgm = tmp_path / "t.pgm"
    pgm.write_bytes(b"P2\n2 2\n255\n")
    r = run("decompose", pgm)
    assert r.returncode == 2 and "not a binary PGM (magic 'P2', expected P5)" in r.stderr
    ok = tmp_path / "ok.csv"
    ok.write_text("a\n1\n2\n3\n4\n5\n")
    r = run("decompose", ok, "--d", "0")
    assert r.returncode == 2 and r.stderr.strip() == "error: --d must be a positive integer or 'auto', got '0'"
    r = run("decompose", ok, "--algo", "vmd")
    assert r.returncode == 2 and "unknown algorithm 'vmd'" in r.stderr


@pytest.mark.gpu
def test_decompose_outputs_byte_identical(cli, gold, tmp_path):
    run("synth", "signals", "--out", tmp_path)
    make_inputs(str(tmp_path))
    for i, case in enumerate(gold["cases"]):
        od = tmp_path / f"out{i}"
        args = []
        for k, v in case["args"].items():
            args += ["--" + k, v]
        r = run("decompose", tmp_path / case["input"], *args, "--out", od)
        assert r.returncode == 0, r.stderr
        got = {f: sha_file(od / f) for f in sorted(os.listdir(od))}
        assert got == case["files"], (i, case["args"])
