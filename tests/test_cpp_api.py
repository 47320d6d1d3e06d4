"""The C++ host API (include/gridshift/gridshift.hpp) end to end: tests/cpp/api_check.cpp is
compiled against libgridshift_cuda.so and its results are compared with the CPU oracle
(bit-exact), and the contract violations must raise the errors.hpp exception types."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2206_02200_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "api_check")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "api_check.cpp"), "-L", LIB,
                    "-lgridshift_cuda", f"-Wl,-rpath,{LIB}", "-o", exe], check=True)
    return exe


def test_cpp_api_compiles(tmp_path):
    # CPU: the header and the library link (no device needed to build)
    _build(tmp_path)


@pytest.mark.gpu
def test_cpp_api_matches_oracle(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    rec = {j["what"]: j for j in (json.loads(line) for line in out.splitlines() if line.strip())}
    X = np.array(rec["points"]["X"]).reshape(-1, 2)
    o = O.run(X, 0.1, 300, O.BUILD_FIXED)
    assert rec["run"]["labels"] == o["labels"].tolist()
    assert np.array_equal(np.array(rec["run"]["centroids"]), o["centroids"].ravel())
    m = O.mspp(X, 0.1, 1e-7, 300)
    assert rec["mspp"]["labels"] == m["labels"].tolist()
    assert np.array_equal(np.array(rec["mspp"]["centroids"]), m["centroids"].ravel())
    t = O.tune(X, [0.05, 0.1, 0.2, 0.4], 300, 200, 7, O.BUILD_FIXED)
    assert rec["tune"]["best_h"] == t["best_h"]
    assert rec["tune"]["scores"] == [s if v else -9.0 for s, v in zip(t["scores"], t["valid"])]
    T, H, W = 8, 96, 128
    fr = np.empty((T, H, W, 3), np.uint8)
    fr[...] = (20, 20, 200)
    for k in range(T):
        fr[k, 30 + k:46 + k, 30 + 3 * k:46 + 3 * k] = (220, 20, 20)
    tr = O.track(fr, [37.5, 37.5, 20.0, 20.0], 0.1)
    assert np.array_equal(np.array(rec["track"]["windows"]), tr["windows"].ravel())
    assert rec["track"]["lost"] == tr["lost"].astype(int).tolist()
    assert rec["errors"]["ok"] == [1] * 7
