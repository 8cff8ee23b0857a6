"""The C-ABI from plain C++ (tests/native/abi_threads.cpp): the program
compiles and links against libsdv_cuda.so with only include/sdv.h (CPU check),
and on a B200 its concurrent calls (two problems on two threads; eight threads
on one trajectory, the reference's apply_columns pattern) are bitwise equal to
serial calls (-m gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "abi_threads.cpp")
LIBDIR = os.path.join(ROOT, "paper_2401_15758_b200", "_build")


def build(out):
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", "-o", str(out), SRC, f"-L{LIBDIR}", "-lsdv_cuda",
                    f"-Wl,-rpath,{LIBDIR}"], check=True, capture_output=True, text=True)
    return out


def test_abi_threads_program_builds_against_header_only(tmp_path):
    exe = build(tmp_path / "abi_threads")
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_abi_concurrent_calls_bitwise_equal_serial(tmp_path):
    exe = build(tmp_path / "abi_threads")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bitwise equal to serial" in r.stdout and "OK" in r.stdout
