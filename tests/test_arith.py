"""The cheaper bucket / y-mod-S forms of csrc/ph_arith.cuh against the reference formulas
restated with 128-bit integers (bucket_fn.hpp:18-32,66-72; reduce.hpp:38-43): host build of
tests/cpp/test_arith.cpp (no GPU). The same header is compiled into the kernels."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_arith_host(tmp_path):
    exe = tmp_path / "test_arith"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I",
                    os.path.join(ROOT, "paper_2502_15539_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "test_arith.cpp"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe), "4000000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:]
    assert r.stdout.strip().endswith("OK (0 failures)")
