"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/rdfft.h declares, and rejects invalid arguments with the documented
status codes before touching the GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rdfft.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2511_01385_b200 import build, rdfft

    build.build()
    return rdfft._lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*([a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ["rdfft_fwd", "rdfft_inv", "rdfft_packed_mul", "rdfft_packed_conjmul", "bca_fwd", "bca_fwd_accum", "bca_bwd"]:
        assert f in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    from paper_2511_01385_b200 import rdfft

    assert set(rdfft.EXPORTS) == set(declared_functions())
    assert lib.rdfft_abi_version() == 104


def test_status_strings(lib):
    for s in range(8):
        assert lib.rdfft_status_str(s)
    assert lib.rdfft_status_str(0) == b"ok"


FAKE = ctypes.c_void_p(0x10000)          # 16-byte aligned, never dereferenced on error paths
FAKE2 = ctypes.c_void_p(0x20000000)
MIS = ctypes.c_void_p(0x10008)


def test_transform_validation(lib):
    for fn in (lib.rdfft_fwd, lib.rdfft_inv):
        assert fn(FAKE, 4, 3, 0, None) == 1        # E_SIZE: not a power of two
        assert fn(FAKE, 4, 1, 0, None) == 1        # E_SIZE: n = 1
        assert fn(FAKE, 4, 131072, 0, None) == 1   # E_SIZE: above 65536
        assert fn(FAKE, 4, 8, 7, None) == 4        # E_DTYPE
        assert fn(FAKE, -1, 8, 0, None) == 5       # E_SHAPE
        assert fn(None, 4, 8, 0, None) == 2        # E_NULL
        assert fn(MIS, 4, 8, 0, None) == 3         # E_ALIGN
        assert fn(None, 0, 8, 1, None) == 0        # batch 0: no-op


def test_packed_validation(lib):
    for fn in (lib.rdfft_packed_mul, lib.rdfft_packed_conjmul):
        assert fn(FAKE, FAKE2, 4, 8, 2, 0, None) == 5   # b_batch not in {1, batch}
        assert fn(FAKE, None, 4, 8, 1, 0, None) == 2
        assert fn(FAKE, ctypes.c_void_p(0x10010), 4, 8, 1, 0, None) == 6  # b inside a
        assert fn(FAKE, FAKE2, 4, 6, 1, 0, None) == 1
        assert fn(FAKE, FAKE2, 0, 8, 1, 0, None) == 0


def test_utility_validation(lib):
    far = ctypes.c_void_p(0x40000000)
    for fn in (lib.rdfft_decode, lib.rdfft_encode):
        assert fn(FAKE, far, 4, 12, 0, None) == 1              # E_SIZE
        assert fn(FAKE, far, 4, 8, 9, None) == 4               # E_DTYPE
        assert fn(FAKE, None, 4, 8, 0, None) == 2              # E_NULL
        assert fn(FAKE, MIS, 4, 8, 0, None) == 3               # E_ALIGN
        assert fn(FAKE, ctypes.c_void_p(0x10020), 4, 8, 0, None) == 6  # overlap (out of place only)
        assert fn(None, None, 0, 8, 0, None) == 0
    assert lib.rdfft_packed_conj(FAKE, 4, 6, 0, None) == 1
    assert lib.rdfft_packed_conj(MIS, 4, 8, 0, None) == 3
    assert lib.rdfft_packed_conj(None, 0, 8, 0, None) == 0
    axpy = lib.rdfft_packed_axpy
    assert axpy(FAKE, far, ctypes.c_float(1.0), 4, 8, 2, 0, None) == 5       # x_batch not in {1, batch}
    assert axpy(FAKE, ctypes.c_void_p(0x10010), ctypes.c_float(1.0), 4, 8, 1, 0, None) == 6
    assert axpy(FAKE, None, ctypes.c_float(1.0), 4, 8, 1, 0, None) == 2
    assert axpy(FAKE, far, ctypes.c_float(1.0), 0, 8, 1, 0, None) == 0


def test_bca_validation(lib):
    y = ctypes.c_void_p(0x40000000)
    assert lib.bca_fwd(FAKE, FAKE2, y, 4, 768, 768, 100, 1, None) == 1      # p not pow2
    assert lib.bca_fwd(FAKE, FAKE2, y, 4, 8192, 8192, 8192, 1, None) == 1   # p above 4096
    assert lib.bca_fwd(FAKE, FAKE2, y, 4, 770, 768, 256, 1, None) == 5      # d_in % p
    assert lib.bca_fwd(FAKE, FAKE2, y, 4, 768, 768, 256, 3, None) == 4      # dtype
    assert lib.bca_fwd(FAKE, FAKE2, None, 4, 768, 768, 256, 1, None) == 2   # y null
    assert lib.bca_fwd(FAKE, FAKE2, ctypes.c_void_p(0x10100), 4, 768, 768, 256, 1, None) == 6  # y overlaps x
    dw = ctypes.c_void_p(0x50000000)
    dx = ctypes.c_void_p(0x60000000)
    # dx may alias g only when d_in == d_out
    g = ctypes.c_void_p(0x70000000)
    assert lib.bca_bwd(FAKE, FAKE2, g, g, dw, 4, 512, 768, 256, 1, None) == 6
    assert lib.bca_bwd(FAKE, FAKE2, g, FAKE, dw, 4, 768, 768, 256, 1, None) == 6   # dx overlaps x
    assert lib.bca_bwd(FAKE, FAKE2, g, dx, None, 4, 768, 768, 256, 1, None) == 2
    assert lib.bca_bwd(FAKE, FAKE2, g, dx, ctypes.c_void_p(0x70000010), 4, 768, 768, 256, 1, None) == 6
    for f in (lib.bca_bwd, lib.bca_bwd_accum):  # the accumulate entry point validates identically
        assert f(FAKE, FAKE2, g, g, dw, 4, 512, 768, 256, 1, None) == 6
        assert f(FAKE, FAKE2, g, dx, None, 4, 768, 768, 256, 1, None) == 2
        assert f(FAKE, FAKE2, g, dx, dw, 4, 768, 768, 100, 1, None) == 1


def test_oracle_not_imported_by_product_path():
    # The product package must never import the oracle (shares no code with it).
    pkg = os.path.join(ROOT, "paper_2511_01385_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b|#include\s+[<\"].*oracle", src, flags=re.M), f


def test_filter_host_validation(lib):
    h = ctypes.c_void_p(0x1000000)
    work = ctypes.c_void_p(0x40000000)
    f = lib.rdfft_filter_host
    assert f(h, 4, 12, 0, None, 0, work, 4, None, None) == 1        # E_SIZE
    assert f(h, 4, 8, 5, None, 0, work, 4, None, None) == 4         # E_DTYPE
    assert f(h, 4, 8, 0, None, 0, work, 1, None, None) == 5         # work_rows < 2
    assert f(h, -1, 8, 0, None, 0, work, 4, None, None) == 5        # negative batch
    assert f(None, 4, 8, 0, None, 0, work, 4, None, None) == 2      # E_NULL (host)
    assert f(h, 4, 8, 0, None, 0, None, 4, None, None) == 2         # E_NULL (work)
    assert f(h, 4, 8, 0, None, 0, MIS, 4, None, None) == 3          # E_ALIGN
    assert f(h, 4, 8, 0, ctypes.c_void_p(0x40000010), 0, work, 4, None, None) == 6  # filt inside work
    assert f(None, 0, 8, 0, None, 0, None, 4, None, None) == 0      # batch 0: no-op


def test_library_objects_call_no_allocator(lib):
    """Zero intermediate allocation (north star), checked on what the library's own object
    files can call: every CUDA / C runtime symbol they import is on an allowlist that holds no
    allocator (no cudaMalloc*, cudaMallocAsync, cudaHostAlloc, cuMemAlloc*, cuMemCreate, malloc,
    operator new).  The GPU test test_zero_allocation checks the same at run time through
    cudaMemGetInfo and torch's allocator."""
    import glob
    import subprocess

    objs = glob.glob(os.path.join(ROOT, "paper_2511_01385_b200", "build", "*.o"))
    assert objs, "build/*.o missing (built by build.build())"
    allowed = {"cudaDeviceGetAttribute", "cudaFuncSetAttribute", "cudaGetDevice", "cudaGetLastError",
               "cudaLaunchKernel", "cudaLaunchKernelExC", "cudaMemsetAsync", "cudaMemcpyAsync",
               "cudaOccupancyMaxActiveBlocksPerMultiprocessorWithFlags", "__cudaPopCallConfiguration",
               "__cudaPushCallConfiguration", "__cudaRegisterFatBinary", "__cudaRegisterFatBinaryEnd",
               "__cudaRegisterFunction", "__cudaRegisterVar", "__cudaUnregisterFatBinary", "_GLOBAL_OFFSET_TABLE_",
               "__cxa_guard_acquire", "__cxa_guard_release", "__fprintf_chk", "__stack_chk_fail", "atexit",
               "getenv", "stderr"}
    seen = set()
    for obj in objs:
        out = subprocess.run(["nm", "-u", obj], capture_output=True, text=True, check=True).stdout
        for line in out.splitlines():
            sym = line.split()[-1]
            if sym.startswith("_Z"):
                dem = subprocess.run(["c++filt", sym], capture_output=True, text=True).stdout.strip()
                assert not re.search(r"operator new|malloc|alloc", dem), (obj, dem)
                continue
            seen.add(sym)
    bad = {s for s in seen if re.search(r"alloc|cuMem|Malloc|HostRegister", s, flags=re.I)}
    assert not bad, bad
    assert seen <= allowed, seen - allowed
