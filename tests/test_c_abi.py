"""The boundary is a C ABI: a plain C99 program (tests/c_abi_smoke.c) including only include/*.h
compiles against libstrata.so and exercises it — argument checks on CPU, a real load with every
engine on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2508_18572_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_2508_18572_b200 import build
    build.build()
    out = str(tmp_path_factory.mktemp("cabi") / "c_abi_smoke")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "c_abi_smoke.c"), "-L", LIBDIR, "-lstrata",
                           f"-Wl,-rpath,{LIBDIR}", "-ldl", "-o", out])
    return out


def test_c_program_cpu_paths(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "c_abi_smoke ok" in r.stdout


@pytest.mark.gpu
def test_c_program_gpu_load(exe):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "c_abi_smoke ok (gpu)" in r.stdout
