"""GridShift hot-path benchmark (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl ours|reference]

A step = one engine.run over one batch of the workload's synthetic input.
`value` is whole-job points/s with the points already resident in HBM (device outputs);
`e2e` is the same metric through the C-ABI with pinned HOST buffers, the H2D copy of the
points and the D2H copy of the labels inside the timed region.  Each timed step is bracketed
by CUDA events on the engine's stream; the L2 is flushed (512 MiB write) before every step.
The default workload is cfg4, the largest single-GPU config: 256 frames of 640 x 480 colour
features.  Under torchrun the 256 frames are split into contiguous frame shards (strong scaling,
no collective on the data path) and the time is the max over ranks.
`--impl reference` times the CPU oracle (the reference algorithm restated, oracle/) on all
host threads instead, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("active-cell updates/sec (cells×iters/s) + end-to-end points/sec; "
          "% HBM roofline")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.rows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [r for r in rows if r[6].isdigit() and int(r[6]) > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in busy for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(int(r[0]) for r in busy),
                "sm_max_mhz": max(int(r[1]) for r in rows), "reasons": reasons,
                "samples": len(busy)}


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def csrc_hash() -> str:
    """Hash of the product kernel sources: a committed ncu traffic figure is only reported for
    the sources it was captured from."""
    import hashlib
    d = os.path.join(ROOT, "paper_2206_02200_b200", "csrc")
    hs = hashlib.sha256()
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".cpp")):
            with open(os.path.join(d, f), "rb") as fh:
                hs.update(f.encode() + fh.read())
    return hs.hexdigest()[:16]


def ncu_traffic(workload: str, kernel: str):
    """dram read+write bytes of one launch of `kernel` from the committed ncu --set full capture
    (profiles/traffic.json, written by scripts/ncu_traffic.py on the GPU box); None when there
    is no capture of the current kernel sources."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t[workload][kernel]
        if e["csrc_hash"] != csrc_hash():
            return None, f"stale: captured from csrc {e['csrc_hash']} ({e['capture']})"
        return int(e["dram_bytes"]), f"{e['capture']} (csrc {e['csrc_hash']})"
    except (OSError, KeyError, ValueError):
        return None, "no capture"


def config_dict(name: str, input_kind: str = "features"):
    """The workload description, identical in both arms (--impl ours / reference)."""
    from paper_2206_02200_b200 import configs as CF
    cfg = CF.CONFIGS[name]
    return {"workload": name, "desc": cfg.desc, "n": cfg.n, "d": cfg.d, "batch": cfg.batch,
            "h": cfg.h, "max_iter": cfg.max_iter,
            "input_dtype": "u8 rgb pixels" if input_kind == "u8" else cfg.dtype}


def workload_input(name: str, rank: int, world: int):
    """This rank's share of the workload.  cfg4: the 256 frames split into contiguous frame
    shards (strong scaling, no collective on the data path); cfg5 under torchrun: a contiguous
    point shard of the one cloud; cfg1-3: replicas (each rank its own copy)."""
    from paper_2206_02200_b200 import configs as CF
    from paper_2206_02200_b200.dist import frame_shard, point_shard
    cfg = CF.CONFIGS[name]
    if name == "cfg4":
        f0, cnt = frame_shard(cfg.batch, world, rank)
        return cfg, CF.generate("cfg4", frames=cnt, frame0=f0), "strong"
    if name == "cfg5" and world > 1:
        X = CF.generate(name)
        p0, cnt = point_shard(X.shape[1], world, rank)
        return cfg, np.ascontiguousarray(X[:, p0:p0 + cnt]), "strong"
    if name == "cfg2":  # replicas: each rank its own independent image (seeded per rank)
        return cfg, CF.voronoi_rgb(seed=2208 + 1000 * rank)[None], "weak"
    return cfg, CF.generate(name), "weak"


def oracle_frames(frames, h, max_iter, threads, budget_s=None):
    """Independent oracle runs (SPEC-literal build) of `frames` over `threads` host threads
    (one GridShift run is sequential; ctypes releases the GIL).  Repeats the
    whole set until budget_s is spent (at least once).  Returns (points/s, points, seconds)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as O
    pts, secs = 0, 0.0
    with ThreadPoolExecutor(threads) as ex:
        while True:
            t0 = time.perf_counter()
            list(ex.map(lambda x: O.run(x, h, max_iter, O.BUILD_SPEC), frames))
            secs += time.perf_counter() - t0
            pts += sum(x.shape[0] for x in frames)
            if budget_s is None or secs >= budget_s:
                break
    return pts / secs, pts, secs


def cpu_baseline(name: str, X: np.ndarray, h: float, max_iter: int, budget_s: float = 10.0):
    """The oracle (SPEC-literal build) on this box's host cores over a bounded sample of the
    workload: every frame on all cores (repeated to ~budget_s), plus a 1-core figure."""
    hi = host_info()
    cores = hi["nproc"] or 1
    frames = [np.ascontiguousarray(X[f], np.float64) for f in range(X.shape[0])]
    threads = max(1, min(cores, len(frames)))
    v_all, pts, secs = oracle_frames(frames, h, max_iter, threads, budget_s)
    v_one, pts1, secs1 = oracle_frames(frames[:max(1, min(len(frames), 8))], h, max_iter, 1)
    return {"value": v_all, "unit": "points/s", "cores": threads, "kind": "port",
            "sample": f"{name}: {len(frames)} frame(s) of {X.shape[1]} points as independent "
                      f"oracle runs (SPEC-literal build) on {threads} thread(s), {pts} points in "
                      f"{secs:.1f} s",
            "single_core": {"value": v_one, "points": pts1, "seconds": round(secs1, 2)},
            "host": hi}


def run_reference(args):
    """--impl reference: the CPU oracle (the reference's algorithm; the reference itself has no
    code) on this arm's workload: the same frames, each step all of them as independent runs
    spread over every host thread -- one GridShift run is sequential, so a
    single-cloud workload (cfg5) runs on one thread.  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2206_02200_b200 import configs as CF
    cfg = CF.CONFIGS[args.workload]
    X = CF.generate(args.workload)
    B, n = X.shape[0], X.shape[1]
    frames = [np.ascontiguousarray(X[f], np.float64) for f in range(B)]
    del X
    hi = host_info()
    threads = max(1, min(hi["nproc"] or 1, B))
    step_times = []
    for s in range(args.warmup + args.steps):
        _, _, dt = oracle_frames(frames, cfg.h, cfg.max_iter, threads)
        if s >= args.warmup:
            step_times.append(dt)
    total = sum(step_times)
    value = B * n * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.workload in ("cfg4", "cfg5") else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.workload),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": threads, "kind": "port",
                         "sample": f"per step all {B} frame(s) of {n} points as independent "
                                   f"oracle runs (SPEC-literal build) on {threads} thread(s)",
                         "host": hi},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0

TUNE_GRID = [round(0.05 * i, 2) for i in range(1, 21)]  # SPEC.md:347 default grid
TUNE_CAP, TUNE_SEED, TUNE_MAX_ITER = 10_000, 2206, 100


def run_tune(args):
    """--workload tune: tune_bandwidth over the cfg2 image features with the
    SPEC's default 20-value grid and silhouette_subsampled (cap 10,000).  A step = one whole
    sweep.  value = points x grid values clustered per second (device-resident input), e2e =
    the same through gs_tune_bandwidth from host memory; --impl reference / cpu_baseline = the
    oracle's gso_tune on the host (bounded: the first grid values that fit ~10 s)."""
    from paper_2206_02200_b200 import configs as CF
    X = CF.voronoi_rgb(seed=2208)  # cfg2 (481 x 321, rgb in [0,1])
    n, d = X.shape
    nh = len(TUNE_GRID)
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return 0
        from oracle import oracle as O
        Xd = X.astype(np.float64)
        times = []
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            O.tune(Xd, TUNE_GRID[:4], TUNE_MAX_ITER, TUNE_CAP, TUNE_SEED, O.BUILD_SPEC)
            if s >= args.warmup:
                times.append(time.perf_counter() - t0)
        value = n * 4 * args.steps / sum(times)
        print(json.dumps({
            "impl": "reference", "metric": "bandwidth sweep: points x h values per second",
            "value": value, "unit": "points*h/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps * nh / 4,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "tune", "n": n, "d": d, "grid": nh,
                                            "cap": TUNE_CAP},
            "cpu_baseline": {"value": value, "unit": "points*h/s", "cores": 1, "kind": "port",
                             "sample": "oracle gso_tune over the first 4 grid values per step"},
            "e2e": {"value": value, "unit": "points*h/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return 0
    import torch
    from paper_2206_02200_b200 import gridshift as G
    torch.cuda.set_device(0)
    tuner = G.Tuner(0, max_concurrent=8)
    Xd = torch.from_numpy(X).cuda()
    lib = G.load_library()
    inp_dev = G.GsInput(Xd.data_ptr(), n, d, G.GS_F32, 1, 1, 0)
    hs = np.ascontiguousarray(TUNE_GRID, np.float64)
    out = (G.GsSweepEntry * nh)()
    best = G.C.c_double()

    def sweep_dev():
        tuner._check(lib.gs_tune_bandwidth(tuner._t, G.C.byref(inp_dev), hs.ctypes.data, nh,
                                           TUNE_MAX_ITER, TUNE_CAP, TUNE_SEED, out,
                                           G.C.byref(best)))

    def sweep_host():
        tuner.tune_bandwidth(X, TUNE_GRID, TUNE_MAX_ITER, TUNE_CAP, TUNE_SEED)

    for _ in range(args.warmup):
        sweep_dev()
        sweep_host()
    clocks = ClockSampler(0)
    clocks.start()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sweep_dev()
    torch.cuda.synchronize()
    t_dev = (time.perf_counter() - t0) / args.steps
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sweep_host()
    t_e2e = (time.perf_counter() - t0) / args.steps
    clk = clocks.stop()
    ents = [dict(h=e.h, score=e.score if e.valid else None, k=e.k, iterations=e.iterations)
            for e in out]
    line = {
        "metric": "bandwidth sweep: points x h values per second", "value": n * nh / t_dev,
        "unit": "points*h/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_dev, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "tune", "desc": "cfg2 image features, SPEC.md:347 grid",
                   "n": n, "d": d, "grid": nh, "cap": TUNE_CAP, "seed": TUNE_SEED,
                   "max_iter": TUNE_MAX_ITER, "concurrent_entries": 8,
                   "timing": "host wall clock around the synchronous sweep call"},
        "best_h": best.value, "entries": ents,
        "e2e": {"value": n * nh / t_e2e, "unit": "points*h/s", "ms_per_step": 1e3 * t_e2e,
                "h2d_bytes_per_step": int(X.nbytes), "d2h_bytes_per_step": 0},
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        from oracle import oracle as O
        t0 = time.perf_counter()
        O.tune(X.astype(np.float64), TUNE_GRID[:4], TUNE_MAX_ITER, TUNE_CAP, TUNE_SEED,
               O.BUILD_SPEC)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n * 4 / dt, "unit": "points*h/s", "cores": 1,
                                "kind": "port",
                                "sample": f"oracle gso_tune over the first 4 grid values "
                                          f"({dt:.1f} s, 1 thread)"}
    print(json.dumps(line))
    tuner.close()
    return 0


TRACK_H = 0.08


def track_setup():
    """cfg4's 256 frames as 8-bit pixels and an initial window on frame 0's largest ellipse
    (the most frequent exact colour: ellipses are solid, the background is noisy)."""
    from paper_2206_02200_b200 import configs as CF
    X = CF.ellipse_frames()
    fr = np.clip(np.rint(X.astype(np.float64) * 255.0), 0, 255).astype(np.uint8)
    fr = fr.reshape(X.shape[0], 480, 640, 3)
    f0 = fr[0].reshape(-1, 3)
    packed = (f0[:, 0].astype(np.int64) << 16) | (f0[:, 1].astype(np.int64) << 8) | f0[:, 2]
    vals, cnt = np.unique(packed, return_counts=True)
    sel = np.nonzero(packed == vals[np.argmax(cnt)])[0]
    ys, xs = sel // 640, sel % 640
    win = [float(xs.mean()), float(ys.mean()), 0.8 * float(np.ptp(xs) + 1),
           0.8 * float(np.ptp(ys) + 1)]
    return fr, win


def run_track(args):
    """--workload track: track_sequence over cfg4's 256 frames (640 x 480,
    8-bit), init on frame 0's largest ellipse, h = 0.08, SPEC defaults f = 1, eta = 1,
    max_inner 20.  A step = init + the 255 tracked frames.  value = tracked frames/s with the
    frames in HBM; e2e = the same from host memory (H2D of the frames inside the step)."""
    fr, win = track_setup()
    T = fr.shape[0]
    rank = int(os.environ.get("RANK", "0"))
    metric = "tracker: frames tracked per second"
    if args.impl == "reference":
        if rank != 0:
            return 0
        from oracle import oracle as O
        nfr = 32  # bounded sample: init + 31 frames per step
        times = []
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            O.track(fr[:nfr], win, TRACK_H)
            if s >= args.warmup:
                times.append(time.perf_counter() - t0)
        value = (nfr - 1) * args.steps / sum(times)
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": value, "unit": "frames/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "track", "frames": T, "H": 480, "W": 640, "h": TRACK_H},
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": 1, "kind": "port",
                             "sample": f"oracle gso_track over the first {nfr} frames per step"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return 0
    import torch
    from paper_2206_02200_b200 import gridshift as G
    torch.cuda.set_device(0)
    tr = G.Tracker(0)
    lib = G.load_library()
    fr_host = torch.from_numpy(fr).pin_memory()
    fr_dev = fr_host.cuda()
    cfg = G.TrackerConfig(TRACK_H)
    c = G.GsTrackerConfig(cfg.h, cfg.f, cfg.eta, cfg.max_inner_iters, cfg.engine_max_iter,
                          cfg.top_k, 0, None)
    w0 = G.GsWindow(*win)
    out = (G.GsWindow * (T - 1))()
    lost = np.zeros(T - 1, np.int32)
    inner = np.zeros(T - 1, np.int32)
    fbytes = 480 * 640 * 3

    def step(dev: bool):
        base = fr_dev.data_ptr() if dev else fr_host.data_ptr()
        k = G.C.c_int64()
        tr._check(lib.gs_track_init(tr._t, base, 480, 640, 1 if dev else 0, G.C.byref(w0),
                                    G.C.byref(c), G.C.byref(k)))
        tr._check(lib.gs_track_sequence(tr._t, base + fbytes, T - 1, 1 if dev else 0, out,
                                        lost.ctypes.data, inner.ctypes.data))

    for _ in range(args.warmup):
        step(True)
        step(False)
    clocks = ClockSampler(0)
    clocks.start()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(True)
    t_dev = (time.perf_counter() - t0) / args.steps
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(False)
    t_e2e = (time.perf_counter() - t0) / args.steps
    clk = clocks.stop()
    wins = np.array([[o.ox, o.oy, o.l, o.w] for o in out])
    line = {
        "metric": metric, "value": (T - 1) / t_dev, "unit": "frames/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_dev,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "track", "desc": "cfg4 frames as 8-bit pixels, largest ellipse",
                   "frames": T, "H": 480, "W": 640, "h": TRACK_H, "init_window": win,
                   "timing": "host wall clock around init + the synchronous sequence call"},
        "lost_frames": int(lost.sum()), "mean_inner": float(inner.mean()),
        "final_window": wins[-1].tolist(),
        "e2e": {"value": (T - 1) / t_e2e, "unit": "frames/s", "ms_per_step": 1e3 * t_e2e,
                "h2d_bytes_per_step": int(fr.nbytes), "d2h_bytes_per_step": int(32 * (T - 1))},
        "gpu_launches": 8, "clocks": clk,
    }
    if not args.no_cpu_baseline:
        from oracle import oracle as O
        t0 = time.perf_counter()
        O.track(fr[:32], win, TRACK_H)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": 31 / dt, "unit": "frames/s", "cores": 1, "kind": "port",
                                "sample": f"oracle gso_track, init + 31 frames ({dt:.2f} s)"}
    print(json.dumps(line))
    tr.close()
    return 0


def run_mspp(args):
    """--workload mspp: the MS++ baseline (mspp_run; parallel Jacobi grid
    mean shift) on the cfg2 image, h = 0.08, tol = 1e-6 h, max_iter 300 -- the comparator of
    the reference's speed claims.  value = points/s through gs_mspp_run from
    device-resident points (host wall clock around the synchronous call); e2e = from host
    memory; the engine's own cfg2 line is the default bench."""
    from paper_2206_02200_b200 import configs as CF
    cloud = args.workload == "mspp5"  # the cfg5 cloud: a first grid beyond one CTA (all SMs)
    X = CF.generate("cfg5")[0] if cloud else CF.voronoi_rgb(seed=2208)
    n, d = X.shape
    h = 1.0 if cloud else 0.08
    wl = {"workload": args.workload, "desc": ("cfg5 cloud (64 M points)" if cloud else "cfg2 image")
          + ", MS++ Jacobi baseline", "n": n, "d": d, "h": h, "tol": 1e-6 * h, "max_iter": 300}
    rank = int(os.environ.get("RANK", "0"))
    metric = "MS++ baseline: points/s"
    if args.impl == "reference":
        if rank != 0:
            return 0
        from oracle import oracle as O
        Xd = X.astype(np.float64)
        times = []
        for s in range(args.warmup + args.steps if not cloud else 1):  # (cfg5: one ~1 min run)
            t0 = time.perf_counter()
            O.mspp(Xd, h, tol=1e-6 * h, max_iter=300)
            if s >= args.warmup or cloud:
                times.append(time.perf_counter() - t0)
        value = n * len(times) / sum(times)
        print(json.dumps({
            "impl": "reference", "metric": metric, "value": value, "unit": "points/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": wl,
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": 1, "kind": "port",
                             "sample": "oracle gso_mspp on the whole " +
                                       ("cfg5 cloud, one run" if cloud else "cfg2 image per step")},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return 0
    import torch
    from paper_2206_02200_b200 import gridshift as G
    torch.cuda.set_device(0)
    eng = G.Engine(0)
    lib = G.load_library()
    Xd = torch.from_numpy(X).cuda()
    Xh = torch.from_numpy(X).pin_memory()
    labels = np.zeros(n, np.int32)
    k = np.zeros(1, np.int64)
    it = np.zeros(1, np.int32)
    cv = np.zeros(1, np.int32)
    res = G.GsResult(labels.ctypes.data, k.ctypes.data, it.ctypes.data, cv.ctypes.data)

    def step(dev: bool):
        inp = G.GsInput(Xd.data_ptr() if dev else Xh.data_ptr(), n, d, G.GS_F32, 1,
                        1 if dev else 0, 0)
        eng._check(lib.gs_mspp_run(eng._ctx, G.C.byref(inp), h, 1e-6 * h, 300, G.C.byref(res),
                                   None))

    for _ in range(args.warmup):
        step(True)
        step(False)
    clocks = ClockSampler(0)
    clocks.start()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(True)
    t_dev = (time.perf_counter() - t0) / args.steps
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(False)
    t_e2e = (time.perf_counter() - t0) / args.steps
    clk = clocks.stop()
    line = {
        "metric": metric, "value": n / t_dev, "unit": "points/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_dev,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(wl, timing="host wall clock around the synchronous call"),
        "k": int(k[0]), "iterations": int(it[0]), "converged": bool(cv[0]),
        "e2e": {"value": n / t_e2e, "unit": "points/s", "ms_per_step": 1e3 * t_e2e,
                "h2d_bytes_per_step": int(X.nbytes), "d2h_bytes_per_step": int(4 * n)},
        "gpu_launches": int(eng.stats()["kernel_launches"]), "clocks": clk,
    }
    if not args.no_cpu_baseline:
        from oracle import oracle as O
        Xs = X[: n // 16] if cloud else X  # (cfg5: a 4 M-point prefix, ~10 s)
        t0 = time.perf_counter()
        O.mspp(Xs.astype(np.float64), h, tol=1e-6 * h, max_iter=300)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": len(Xs) / dt, "unit": "points/s", "cores": 1,
                                "kind": "port",
                                "sample": f"oracle gso_mspp, one run on {len(Xs)} points of the "
                                          f"{'cfg5 cloud' if cloud else 'cfg2 image'} ({dt:.2f} s)"}
    print(json.dumps(line))
    eng.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg4",
                    choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "tune", "track", "mspp", "mspp5"],
                    help="default cfg4: the largest single-GPU config (256 frames). tune: the "
                         "bandwidth sweep (SURVEY.md §8(f)2) over the cfg2 image; track: the "
                         "tracker (§8(f)3) over the cfg4 frames; mspp: the MS++ baseline "
                         "(§8(f)4) on the cfg2 image")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--input", default="features", choices=["features", "u8"],
                    help="u8: the image workloads (cfg2, cfg4) as 8-bit RGB pixels, features "
                         "formed on the device (segmentation front end, SURVEY.md §8(f)1)")
    ap.add_argument("--profile-device", action="store_true",
                    help="profiling aid: device-resident steps only (no e2e / phase passes)")
    args = ap.parse_args()
    if args.workload == "tune":
        return run_tune(args)
    if args.workload == "track":
        return run_track(args)
    if args.workload in ("mspp", "mspp5"):
        return run_mspp(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2206_02200_b200 import gridshift as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)  # the engine and the timing events share it
    eng = G.Engine(local, stream.cuda_stream)

    cfg, X, scaling = workload_input(args.workload, rank, world)
    # cfg5 over several GPUs: ONE cloud split into contiguous point shards (dist.run_cloud:
    # partial cells all-gathered, identical iteration on every rank, own points labelled)
    shard_cloud = args.workload == "cfg5" and world > 1
    if shard_cloud:
        from paper_2206_02200_b200.dist import run_cloud
    if args.input == "u8":
        if args.workload not in ("cfg2", "cfg4") or shard_cloud:
            raise SystemExit("--input u8 applies to the image workloads cfg2 and cfg4")
        X = np.clip(np.rint(X.astype(np.float64) * 255.0), 0, 255).astype(np.uint8)
    B, n, d = X.shape
    dt = G.GS_U8 if X.dtype == np.uint8 else (G.GS_F32 if X.dtype == np.float32 else G.GS_F64)
    # timed steps record only the binning kernel's CUDA events (the roofline's kernel time);
    # the per-phase times come from a separate, untimed diagnostic pass (events cost ~30 us)
    econf = G.EngineConfig(cfg.h, cfg.max_iter, debug_flags=G.GS_TIME_KERNEL)
    econf_e2e = G.EngineConfig(cfg.h, cfg.max_iter)
    econf_phases = G.EngineConfig(cfg.h, cfg.max_iter, debug_flags=G.GS_TIME_PHASES)
    X_host = torch.from_numpy(X).pin_memory()
    X_dev = X_host.to(dev)
    labels_dev = torch.empty((B, n), dtype=torch.int32, device=dev)
    labels_host = torch.empty((B, n), dtype=torch.int32).pin_memory()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step(device_resident: bool, conf=None):
        conf = conf or econf
        if shard_cloud:
            run_cloud(eng, X_dev[0] if device_resident else X[0], cfg.h, cfg.max_iter)
            return
        if device_resident:
            eng.run_raw(X_dev.data_ptr(), n, d, dt, B, True, conf, labels_dev.data_ptr(),
                        device_outputs=True)
        else:  # the public call from pinned host memory (frame-group pipeline for batches)
            eng.run_raw(X_host.data_ptr(), n, d, dt, B, False, econf_e2e, labels_host.data_ptr())

    def timed(device_resident: bool, steps: int):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        stats = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for s in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            ev[s][0].record(stream)
            step(device_resident)
            ev[s][1].record(stream)
            stats.append(eng.stats())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = [a.elapsed_time(b) for a, b in ev]
        return ms, stats

    if args.profile_device:  # ncu launch lists / captures of the device-resident step alone
        for _ in range(args.warmup + args.steps):
            step(True)
        torch.cuda.synchronize()
        eng.close()
        return 0
    for _ in range(args.warmup):
        step(True)
        step(False)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ms_dev, st_dev = timed(True, args.steps)
    ms_e2e, st_e2e = timed(False, args.steps)
    clk = clocks.stop()
    st_phase = []  # untimed diagnostic pass with every phase event
    for _ in range(3):
        step(True, econf_phases)
        st_phase.append(eng.stats())
    torch.cuda.synchronize()

    tot_dev, tot_e2e = sum(ms_dev), sum(ms_e2e)
    pts_rank = B * n * args.steps
    if world > 1:
        t = torch.tensor([tot_dev, tot_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_dev, tot_e2e = t.tolist()
        p = torch.tensor([float(pts_rank)], dtype=torch.float64, device=dev)
        dist.all_reduce(p, op=dist.ReduceOp.SUM)
        pts_all = cfg.n * args.steps if shard_cloud else int(p.item())
    else:
        pts_all = pts_rank
    value = pts_all / (tot_dev / 1e3)
    e2e = pts_all / (tot_e2e / 1e3)
    # cells x iterations (Σ m_t) per second over the iteration phase
    s0 = st_dev[-1]
    cells = sum(s["cells_swept"] for s in st_dev)
    it_ms = float(np.mean([s["ms_iterate"] for s in st_phase])) * len(st_dev)
    launches = int(np.median([s["kernel_launches"] for s in st_dev]))
    launches_e2e = int(np.median([s["kernel_launches"] for s in st_e2e]))
    lib_calls = int(np.median([s["lib_calls"] for s in st_dev]))

    # roofline of the n-scale binning kernel K2: algorithmic bytes = points read + slot write
    peak, peak_kind = peaks()
    s_in = {G.GS_F32: 4, G.GS_F64: 8, G.GS_U8: 1}[dt]
    slot_b = int(s0.get("slot_bytes", 4) or 4)
    kbin_ms = float(np.mean([s["ms_k_bin"] for s in st_dev]))
    kbin_bytes = B * n * ((3 if dt == G.GS_U8 else d * s_in) + slot_b)
    kbin_gbs = kbin_bytes / (kbin_ms / 1e3) / 1e9
    phase = {k: float(np.mean([s[k] for s in st_phase]))
             for k in ("ms_bin", "ms_iterate", "ms_label", "ms_k_bin", "ms_k_label")}
    phase["note"] = "untimed diagnostic pass with all phase events; timed steps record K2 only"
    dominant = max(("binning phase (K2+K3)", phase["ms_bin"]),
                   ("iteration phase (K8 / global path)", phase["ms_iterate"]),
                   ("label phase (K7)", phase["ms_label"]), key=lambda x: x[1])[0]
    # whole-step algorithmic bytes: n (d s_in + 4) + Σ m_t (24 + 16 d)
    it_bytes = int(s0["cells_swept"] * (24 + 16 * d))  # B_c = 24 + 16d
    step_bytes = B * n * ((3 if dt == G.GS_U8 else d * s_in) + 4) + it_bytes
    step_ms = tot_dev / args.steps
    if phase["ms_iterate"] >= phase["ms_bin"] and phase["ms_iterate"] > 0:
        ach = it_bytes / (phase["ms_iterate"] / 1e3) / 1e9
        dominant_roofline = {
            "kernel": "k_resident (K8) / global-path sweeps: the iteration phase",
            "bound": "latency (sweep DAG depth x per-level round trips), not hbm",
            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "algorithmic_bytes": it_bytes, "ms": phase["ms_iterate"],
            "note": "sum over the run of m_t x (24 + 16d) bytes / iteration-phase time"}
    else:
        dominant_roofline = {"kernel": "k_bin (K2 binning)", "same_as": "roofline"}
    traffic, traffic_src = (ncu_traffic(args.workload, "k_bin")
                            if not shard_cloud and args.input == "features" else (None, "n/a"))
    out = {
        "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_dict(args.workload, args.input),
        "l2": "flushed (512 MiB write) before every timed step",
        "parallelism": (f"one cloud in {world} point shards (partial cells all-gathered, "
                        f"replicated iteration)") if shard_cloud else
                       (f"{B} of the {cfg.batch} frames on this rank (frame shards x{world})"
                        if args.workload == "cfg4" else f"replicas x{world}"),
        "step_ms_dist": {"min": float(np.min(ms_dev)), "median": float(np.median(ms_dev)),
                         "max": float(np.max(ms_dev)),
                         "e2e_median": float(np.median(ms_e2e))},
        "cell_updates_per_s": cells / (it_ms / 1e3) if it_ms > 0 else None,
        "cells_swept_per_step": s0["cells_swept"], "m0": s0["m0"], "k": s0["k_total"],
        "iterations": s0["max_iterations"],
        "phase_ms": phase, "dominant_phase": dominant,
        "roofline": {"kernel": "k_bin (K2 binning)", "bound": "hbm", "achieved": kbin_gbs,
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": kbin_gbs / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes": kbin_bytes,
                     "bytes_per_point": (3 if dt == G.GS_U8 else d * s_in) + slot_b,
                     "ms": kbin_ms},
        "roofline_step": {"achieved": step_bytes / (step_ms / 1e3) / 1e9, "peak": peak,
                          "unit": "GB/s", "frac": step_bytes / (step_ms / 1e3) / 1e9 / peak,
                          "algorithmic_bytes": step_bytes,
                          "note": "whole step: n (d s_in + 4) + sum_t m_t (24 + 16 d) bytes"},
        "roofline_dominant": dominant_roofline,
        "e2e": {"value": e2e, "unit": "points/s", "h2d_bytes_per_step": int(X.nbytes),
                "d2h_bytes_per_step": int(B * n * 4), "ms_per_step": tot_e2e / args.steps,
                "gpu_launches": launches_e2e,
                "path": "gs_run from pinned host memory" +
                        (" (frame-group pipeline)" if B >= 4 and X.nbytes >= (64 << 20) else "")},
        "gpu_launches": launches, "lib_calls": lib_calls,
        "sweep_modes": s0.get("sweep_modes"), "resident_cycles": s0.get("resident_cycles"),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Xc = X if X.dtype != np.uint8 else X.astype(np.float64) / 255.0
        out["cpu_baseline"] = cpu_baseline(args.workload, Xc, cfg.h, cfg.max_iter,
                                           args.cpu_budget)
    if rank == 0:
        print(json.dumps(out))
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
