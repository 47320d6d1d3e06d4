"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every symbol the
header declares, and validates arguments with the errors.hpp status mapping (no device)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2206_02200_b200 import gridshift as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gridshift_c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_what_python_binds():
    assert declared_symbols() == sorted(G.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = G.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_oracle_not_linked_into_product():
    # the product library must not contain or load the oracle (no CPU fallback)
    data = open(G.LIB_PATH, "rb").read()
    assert b"gso_run" not in data and b"liboracle" not in data


def _validate(n=10, d=2, h=0.5, max_iter=10, batch=1, dtype=G.GS_F64, null=False):
    lib = G.load_library()
    buf = C.c_double(0)
    inp = G.GsInput(None if null else C.addressof(buf), n, d, dtype, batch, 0, 0)
    cfg = G.GsConfig(h, max_iter, 0)
    return lib.gs_validate(C.byref(inp), C.byref(cfg))


def test_validate_status_codes():
    assert _validate() == 0
    assert _validate(h=0.0) == 2           # InvalidBandwidthError SPEC.md:44
    assert _validate(h=-0.5) == 2
    assert _validate(h=float("nan")) == 2
    assert _validate(h=float("inf")) == 2
    assert _validate(n=0) == 3             # EmptyInputError SPEC.md:62
    assert _validate(d=0) == 4             # InvalidParameterError
    assert _validate(d=13) == 4            # SPEC.md:96 d <= 12
    assert _validate(max_iter=0) == 4
    assert _validate(batch=0) == 4
    assert _validate(dtype=7) == 4
    assert _validate(null=True) == 4


def test_python_mirror_raises_reference_types():
    with pytest.raises(G.InvalidBandwidthError):
        G.validate(10, 2, 0.0)
    with pytest.raises(G.EmptyInputError):
        G.validate(0, 2, 0.5)
    with pytest.raises(G.InvalidParameterError):
        G.validate(10, 13, 0.5)
    # hierarchy mirrors errors.hpp:14-28
    assert issubclass(G.InvalidBandwidthError, G.InvalidInputError)
    assert issubclass(G.EmptyInputError, G.InvalidInputError)
    assert issubclass(G.InvalidInputError, G.Error)
    with pytest.raises(G.InvalidBandwidthError):
        G.run(np.zeros((3, 2)), G.EngineConfig(h=0.0))


def test_fixed_shift_matches_oracle():
    from oracle import oracle as O
    for n in (1, 2, 3, 100_000, 154_401, 2_073_600, 307_200, 64_000_000):
        for h in (1e-3, 0.06, 0.08, 0.5, 1.0, 7.5, 1e6):
            assert G.fixed_shift(n, h) == O.fixed_shift(n, h)


def test_status_strings():
    lib = G.load_library()
    for s in range(11):
        assert lib.gs_status_string(s)


def test_no_device_is_loud():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(G.Error):
        G.Engine(0)


def test_cmake_project_configures(tmp_path):
    """The CMake build (CMakeLists.txt: CUDA language, sm_100a only, the gridshift::cuda target a
    reference-side CMake links) configures with the toolchain in this image; the full build is
    the same sources and flags as the Makefile's and is not repeated here."""
    import shutil
    import subprocess
    cmake = shutil.which("cmake")
    if cmake is None or not os.path.exists("/usr/local/cuda/bin/nvcc"):
        pytest.skip("cmake or nvcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([cmake, "-S", root, "-B", str(tmp_path), "-G", "Ninja"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    ninja = (tmp_path / "build.ninja").read_text()
    assert "libgridshift_cuda.so" in ninja and "sm_100a" in ninja and "--fmad=false" in ninja
