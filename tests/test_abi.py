"""CPU-only: the C-ABI library loads and exports every entry point declared
in include/*.h (no device calls)."""
import ctypes
import glob
import os
import re

from paper_1805_11144_b200 import engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(neng_\w+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_headers_declare_the_engine_surface():
    names = declared_functions()
    for required in ("neng_gpu_create", "neng_gpu_run", "neng_gpu_reset", "neng_gpu_read_signal",
                     "neng_gpu_buffer_storage", "neng_gpu_steps_completed", "neng_gpu_destroy",
                     "neng_gpu_last_error", "neng_run_passes"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = engine.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    so = engine.LIB_PATH
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_no_contracted_paired_fma_in_sass():
    """Bit parity needs every product rounded before its sum.  The kernels are
    built with -fmad=false, but ptxas still contracts a paired multiply feeding
    a paired add (mul.rn.f32x2 -> add.rn.f32x2) into FFMA2, so the code never
    chains them; this keeps it that way."""
    import shutil
    import subprocess

    import pytest

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", engine.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "fused_run_kernel" in sass
    # the kernels' paired products are fma(a, b, -0) with the (-0, -0) pair in a
    # uniform register (a kernel parameter): any other addend is a contraction
    ffma2 = re.findall(r"FFMA2 [^;]*;", sass)
    bad = [f for f in ffma2 if not re.search(r",\s*-?UR\d+(\.F32x2\.HI_LO)?\s*;", f)]
    assert not bad, bad[:4]


def test_no_odd_uniform_memory_descriptors_in_sass():
    """A 64-bit memory descriptor lives in an even/odd uniform register pair.
    ptxas 12.9 emitted `LDGSTS ... desc[UR1]` for the cp.async with an
    L2::cache_hint operand in some kernel instances, which faulted at run time
    with "illegal instruction" (the round-1 "code-placement sensitive" fault).
    The kernels no longer use that form; this keeps every descriptor even."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", engine.LIB_PATH], capture_output=True, text=True, check=True).stdout
    # memory descriptors only (tcgen05's idesc/gdesc operands are other register kinds)
    odd = re.findall(r"^.*[\s,]desc\[UR\d*[13579]\].*$", sass, flags=re.M)
    assert not odd, odd[:4]


def test_bad_arguments_fail_with_status_not_crash():
    lib = engine.lib()
    out = ctypes.c_void_p()
    assert lib.neng_gpu_create(None, 1, 1, None, ctypes.byref(out)) == 6  # NENG_INVALID_ARGUMENT
    assert b"null" in lib.neng_last_error()
