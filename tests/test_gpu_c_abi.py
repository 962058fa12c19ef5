"""The C ABI from plain C (tests/c_abi/abi_smoke.c): built with gcc against
include/lasgd_sync.h and the in-tree library, run on the GPU, bit-exact checks inside."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plain_c_consumer(tmp_path):
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    lib = os.path.join(ROOT, "paper_2203_13085_b200", "_lib")
    exe = str(tmp_path / "abi_smoke")
    subprocess.run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(cuda, "include"), os.path.join(ROOT, "tests", "c_abi", "abi_smoke.c"),
                    "-L", lib, "-llasgd_sync", "-L", os.path.join(cuda, "lib64"), "-lcudart", "-o", exe],
                   check=True)
    env = dict(os.environ, LD_LIBRARY_PATH=lib + ":" + os.path.join(cuda, "lib64") + ":"
               + os.environ.get("LD_LIBRARY_PATH", ""))
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "c abi ok" in r.stdout
