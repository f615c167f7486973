"""Run-time allocation counter (the library allocates no device or host memory per call;
S:L185).  tools/alloc_count.cu subscribes to every CUDA driver and runtime API call through CUPTI and
counts the allocator calls (cuMemAlloc*, cuMemCreate, cuMemHostAlloc, cudaMalloc*, ...) made while
every C-ABI entry point runs — first (cold) calls and repeated (warm) calls, every transform size
and both dtypes, every BCA kernel family, the host-buffer pipeline.  The static check of the
library's imported symbols is tests/test_abi_cpu.py::test_library_objects_call_no_allocator."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"
TGT = os.path.join(CUDA, "targets", "x86_64-linux")


def test_no_allocation_through_cupti(tmp_path, cuda_device):
    from paper_2511_01385_b200 import build

    lib = build.build()
    exe = str(tmp_path / "alloc_count")
    subprocess.run([os.path.join(CUDA, "bin", "nvcc"), "-O2", "-std=c++17", "-o", exe,
                    os.path.join(ROOT, "tools", "alloc_count.cu"), "-I", os.path.join(TGT, "include"),
                    "-L", os.path.join(TGT, "lib"), "-lcupti", "-ldl"], check=True, capture_output=True)
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = os.path.join(TGT, "lib") + ":" + env.get("LD_LIBRARY_PATH", "")
    out = subprocess.run([exe, lib], capture_output=True, text=True, env=env, timeout=600)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else ""
    assert line, out.stderr
    rep = json.loads(line)
    assert rep["status_or"] == 0, rep
    assert rep["cold_api_calls"] > 0 and rep["warm_api_calls"] > 0, rep  # the subscriber saw the calls
    assert rep["cold_allocs"] == 0, rep["cold_alloc_names"]
    assert rep["warm_allocs"] == 0, rep["warm_alloc_names"]
    assert out.returncode == 0, out.stderr
