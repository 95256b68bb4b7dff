"""The device noise path's restatement of glibc's log and sincos (paper_2106_15319_b200/csrc/
semd_libm.cuh, the functions k_box_muller runs) against the system libm, bit for bit, on the
white_noise input distribution plus edge sweeps of every branch (tests/cpp/libm_check.cpp).
This is what makes the device's Box-Muller equal to the reference's (emd.cpp:189-198)."""
import os
import subprocess

from tests.conftest import ROOT


def test_libm_restatement_bit_exact(tmp_path):
    exe = str(tmp_path / "libm_check")
    src = os.path.join(ROOT, "tests", "cpp", "libm_check.cpp")
    inc = os.path.join(ROOT, "paper_2106_15319_b200", "csrc")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-mfma", "-I" + inc, src, "-o", exe, "-lm"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for seed in (1, 2106):
        r = subprocess.run([exe, "10000000", str(seed)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.strip().startswith("mismatches 0 0 0"), r.stdout


def test_tables_match_installed_libm(tmp_path):
    """The generated table header is what gen_libm_tables.py reads from this image's libm."""
    import importlib.util
    gen = os.path.join(ROOT, "paper_2106_15319_b200", "csrc", "gen_libm_tables.py")
    spec = importlib.util.spec_from_file_location("gen_libm_tables", gen)
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    committed = open(m.OUT).read()
    m.OUT = str(tmp_path / "t.h")
    m.main()
    assert open(m.OUT).read() == committed
