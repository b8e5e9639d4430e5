"""C++ tests through include/snap.hpp (the C++ mirror of the reference API), compiled with
g++ -std=c++20 against libsnap.so: allocator tests on CPU, device tests on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2202_07848_b200")


def build_and_run(name, tmp_path):
    exe = str(tmp_path / name)
    src = os.path.join(ROOT, "tests", "cpp", f"{name}.cpp")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(ROOT, "tests", "cpp"), src, "-o", exe,
                    f"-L{LIBDIR}", "-lsnap", f"-Wl,-rpath,{LIBDIR}"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    return r


def test_cpp_alloc(snap, tmp_path):
    r = build_and_run("test_alloc", tmp_path)
    assert r.returncode == 0, r.stdout


@pytest.mark.gpu
def test_cpp_device(snap, tmp_path):
    r = build_and_run("test_device", tmp_path)
    assert r.returncode == 0, r.stdout
