"""CPU checks of the drop-in boundary: libpolycast_cuda.so loads, exports every
symbol include/polycast_cuda.h declares, targets sm_100a, and refuses to run
without a GPU (no CPU fallback)."""
import os
import re
import subprocess

import pytest

from paper_2306_04316_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "polycast_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert {"pc_create", "pc_classify", "pc_classify_csr", "pc_count_crossings", "pc_classify_dev",
            "pc_classify_csr_dev", "pc_destroy", "pc_last_error"} <= set(syms)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, f"{s} has no ctypes signature"
    out = subprocess.run(["nm", "-D", "--defined-only", _native.CUDA_LIB], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.CUDA_LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_fma_in_c1_kernels():
    """Rule P1: no DFMA in the division-free C1 kernels (C2/Robust divisions use the
    correctly rounded __ddiv_rn sequence, which contains DFMA internally)."""
    sass = subprocess.run(["cuobjdump", "-sass", _native.CUDA_LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    c1 = [f for f in funcs if re.match(r"\S*(pip_tile_kernelILi0E|pip_csr_warp_kernelILi0E|pip_csr_tile_kernelILi0E|count_kernelILi0E)", f)]
    assert len(c1) >= 3
    for f in c1:
        assert "DFMA" not in f


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="GPU present")
def test_no_cpu_fallback_without_gpu():
    from paper_2306_04316_b200 import DeviceError, Engine
    with pytest.raises(DeviceError):
        Engine()


def test_cpp_api_compiles_against_header(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include <polycast/polycast.hpp>\nint main(){ polycast::PointBatch b; '
                   'polycast::Polygon p(polycast::Ring({{0,0},{1,0},{1,1},{0,0}}));'
                   'return (int)polycast::classify_batch(b, p, polycast::CrossingMode::C1).verdicts.size(); }\n')
    r = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
