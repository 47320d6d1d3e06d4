"""Writes tests/golden/spec_kats.json: the known-answer examples of the reference spec.

The reference ships no test files or golden outputs; its only pinned
answers are the [TRIVIAL]/[DERIVED] examples in /root/reference/SPEC.md.  Each entry below
transcribes one of them with its SPEC line.  Expected values are the SPEC's own numbers;
`tol` is the comparison tolerance where the SPEC states a real-number result.

Run:  python tests/golden/make_spec_kats.py
"""
import json
import os

KATS = {
    "grid_index": [
        {"x": [2.5, 0.3], "h": 1.0, "key": [2, 0], "src": "SPEC.md:46"},
        {"x": [-0.3], "h": 0.5, "key": [-1], "src": "SPEC.md:47"},
        {"x": [0.78, 0.78], "h": 0.78, "key": [1, 1], "src": "SPEC.md:48"},
    ],
    "neighborhood": [
        {"d": 1, "j": [5], "expect": [[4], [5], [6]], "src": "SPEC.md:55"},
        {"d": 2, "j": [0, 0], "count": 9, "src": "SPEC.md:56"},
        {"d": 3, "j": [7, -2, 4], "count": 27, "src": "SPEC.md:57"},
    ],
    "build": [
        {"X": [[0.1], [0.2], [0.9]], "h": 0.5, "keys": [[0], [1]], "counts": [2, 1],
         "centroids": [[0.15], [0.9]], "tol": 1e-12, "src": "SPEC.md:64"},
        {"X": [[0.3, -1.7]], "h": 0.25, "keys": [[1, -7]], "counts": [1],
         "centroids": [[0.3, -1.7]], "tol": 1e-12, "src": "SPEC.md:65"},
        {"X": [[0.42, 0.17, 0.9]] * 7, "h": 0.1, "keys": [[4, 1, 9]], "counts": [7],
         "centroids": [[0.42, 0.17, 0.9]], "tol": 1e-12, "src": "SPEC.md:66"},
    ],
    # merge_into exercised through iterate_once on isolated cells whose centroids rehome to one
    # key: the sweep leaves them unchanged and the rehome merges them in visit
    # order (SPEC.md:120(d), :67-75).
    "merge": [
        {"keys": [[-10], [10]], "counts": [1, 3], "centroids": [[2.25], [2.75]], "h": 1.0,
         "out_keys": [[2]], "out_counts": [4], "out_centroids": [[(2.25 + 3 * 2.75) / 4]],
         "tol": 1e-12, "src": "SPEC.md:73"},
        {"keys": [[-10], [10], [20]], "counts": [2, 1, 1], "centroids": [[0.0], [0.4], [0.8]],
         "h": 1.0, "out_keys": [[0]], "out_counts": [4], "out_centroids": [[0.3]],
         "tol": 1e-12, "src": "SPEC.md:75"},
    ],
    "iterate_once": [
        {"keys": [[0], [1]], "counts": [3, 1], "centroids": [[0.4], [0.6]], "h": 0.5,
         "swept": [[0.45], [0.4875]], "out_keys": [[0]], "out_counts": [4],
         "out_centroids": [[0.459375]], "changed": True, "tol": 1e-15, "src": "SPEC.md:123"},
        {"keys": [[3]], "counts": [5], "centroids": [[1.7]], "h": 0.5, "swept": [[1.7]],
         "out_keys": [[3]], "out_counts": [5], "out_centroids": [[1.7]], "changed": False,
         "tol": 0.0, "src": "SPEC.md:124"},
        {"keys": [[0], [5]], "counts": [2, 3], "centroids": [[0.2], [2.6]], "h": 0.5,
         "swept": [[0.2], [2.6]], "out_keys": [[0], [5]], "out_counts": [2, 3],
         "out_centroids": [[0.2], [2.6]], "changed": False, "tol": 0.0, "src": "SPEC.md:125"},
    ],
    "has_converged": [
        {"keys": [[0]], "expect": True, "src": "SPEC.md:132"},
        {"keys": [[0], [1]], "expect": False, "src": "SPEC.md:133"},
        {"keys": [[0], [3]], "expect": True, "src": "SPEC.md:134"},
    ],
    "run": [
        {"X": [[0.11], [0.12], [0.13], [0.14], [0.15]], "h": 0.5, "k": 1, "iterations": 1,
         "labels": [0, 0, 0, 0, 0], "centroids": [[0.13]], "tol": 1e-12, "src": "SPEC.md:141"},
        {"X": [[0.1, 0.2], [0.15, 0.25], [0.12, 0.22], [5.0, 6.0], [5.1, 6.1]], "h": 0.5,
         "k": 2, "labels": [0, 0, 0, 1, 1],
         "centroids": [[(0.1 + 0.15 + 0.12) / 3, (0.2 + 0.25 + 0.22) / 3], [5.05, 6.05]],
         "tol": 1e-12, "src": "SPEC.md:142"},
    ],
    "run_traced": [
        {"X": [[0.3, 0.3, 0.3]], "h": 1.0, "snapshots": 1, "src": "SPEC.md:152"},
    ],
    # the engine's sequential semantics, NOT the parallel MS++ update (SPEC.md:205 contrast)
    "jacobi_contrast": [
        {"keys": [[0], [1]], "counts": [3, 1], "centroids": [[0.4], [0.6]], "h": 0.5,
         "engine_cell1": 0.4875, "jacobi_cell1": 0.45, "src": "SPEC.md:205"},
    ],
    "errors": [
        {"case": "h_zero", "h": 0.0, "error": "InvalidBandwidthError", "src": "SPEC.md:44"},
        {"case": "h_negative", "h": -1.0, "error": "InvalidBandwidthError", "src": "SPEC.md:44"},
        {"case": "empty", "n": 0, "error": "EmptyInputError", "src": "SPEC.md:62"},
        {"case": "nan", "error": "InvalidInputError", "src": "SPEC.md:24, :44"},
    ],
}

if __name__ == "__main__":
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_kats.json")
    with open(path, "w") as f:
        json.dump(KATS, f, indent=1)
    print("wrote", path)
