#!/usr/bin/env python
"""Benchmark: Mrays/s (transmittance + scattering) of the Gabor Fields hot path on B200, and the
fraction of the HBM roofline of the dominant kernel.

Default workload (BASELINE.json configs[4], "config 5", the configuration the metric's "at 1/2/4/8
B200" is quoted on): the 3,993,600-primitive army of bunny-like assets, 4096x4096, multiple scattering
depth 8, LOD sweep = 5 frames per step (4 global static masks {0}, {0,1}, {0..2}, {0..3} and the
distance-banded mask of fig:army_bunny: near all levels, mid 0..2, far 0..1), 1 spp per frame.  At N
GPUs every rank renders its 32x32 tiles of every frame (tile t -> rank t mod N, scene replicated,
strong scaling: the frame is fixed) and one NCCL reduce per frame gathers the image on rank 0 (the
tiles are disjoint).  A "ray" is one ray query: camera, extension (free-flight) or NEE shadow ray.
`--config 1..4` selects the other configurations (config 4: the 1M-primitive HBM question).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 1..5]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2602_05081_b200 import inputs as I  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP32 algorithmic work model per unit: node box test, primitive whitening test, hit
# setup, one complex-erf endpoint (Horner, 30 complex terms, 4 FFMA = 8 FLOP each), real erf.
ERF_TERMS = 30
FLOP_NODE, FLOP_TEST, FLOP_HIT, FLOP_ERF = 24, 45, 40, 8 * ERF_TERMS
FLOP_ERF_REAL = 20
FLOP_ROOT_EVAL = 20
# Algorithmic bytes per unit (B_ray = 32 + 8 + 64 N_v + 64 N_t, uncached): a ray's 32-byte
# origin/direction/range and 8-byte result, 32 bytes per node box test (a visited node is a 64-byte
# child pair, counted as 2 box tests), 64 bytes per primitive record tested.
BYTES_RAY, BYTES_NODE, BYTES_TEST = 40, 32, 64
DEFAULT_CONFIG = 5


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.samples, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and "Active" == s[3 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def replica_check(h, dist, device):
    """SURVEY §8(e) replica check: True iff the 64-bit BVH hash h is equal on every rank (all-reduce MIN
    and MAX of its two 32-bit halves)."""
    import torch
    v = torch.tensor([h & 0xFFFFFFFF, h >> 32], dtype=torch.int64, device=device)
    lo, hi = v.clone(), v.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    return bool(torch.equal(lo, hi))


def load_traffic(config, stage):
    """(kernel, DRAM bytes per launch, source) of the stage's kernel from the committed ncu --set full
    capture of this round, or Nones."""
    for fn in ("r02_traffic.json",):
        try:
            t = json.load(open(os.path.join(ROOT, "profiles", fn)))
            e = t[f"cfg{config}"][stage]
            return e["kernel"], e["dram_bytes_per_launch"], "profiles/" + fn
        except (OSError, KeyError, ValueError):
            continue
    return None, None, None


def load_peaks():
    try:
        return json.load(open(PEAKS_FILE))
    except OSError:
        return {}


def workload(config):
    if config == 1:
        sc = I.scene_cfg1()
        descs = [I.render_desc_cfg1()]
        name = "cfg1: 1k random Gabor primitives, 64x64, 1 spp primary-ray transmittance (tomography), full LOD"
    elif config == 2:
        sc = I.scene_cfg2()
        descs = [I.render_desc_cfg2(i) for i in range(4)]
        name = ("cfg2: bunny-like 100k-primitive Gabor field, 1024x1024, single scattering, 4 static LOD levels "
                "({0},{0,1},{0..2},{0..3}), 1 spp per level")
    elif config == 3:
        sc = I.scene_cfg3()
        descs = [I.render_desc_cfg3()]
        name = ("cfg3: procedural clouds, 327,600 primitives (15,600 Gaussian cores + 312,000 Gabors), 1024x1024, "
                "multiple scattering depth 8, full LOD, 1 spp")
    elif config == 4:
        sc = I.scene_cfg4()
        descs = [I.render_desc_cfg4()]
        name = ("cfg4: dense 1M-primitive asset, 2048x2048, multiple scattering depth 8, stochastic per-recursion "
                "masks (PL+CV Accum. beta 0.2 x orientation Importance, Zero NEE), 1 spp")
    else:
        sc = I.scene_cfg5()
        descs = [I.render_desc_cfg5(lv) for lv in ((0,), (0, 1), (0, 1, 2), (0, 1, 2, 3), "banded")]
        name = ("cfg5: 3,993,600-primitive army (120 x 33,280-primitive bunny-like assets, 3 distance bands), "
                "4096x4096, multiple scattering depth 8, LOD sweep: 4 global static masks ({0},{0,1},{0..2},{0..3}) "
                "+ the distance-banded mask (near 0..3, mid 0..2, far 0..1), 1 spp per frame")
    return sc, descs, name


# ----------------------------------------------------------------------------------------------
ORACLE_PATHS = {1: 4096, 2: 4096, 3: 512, 4: 96, 5: 64}  # oracle sample per step (a few seconds of CPU)


def cpu_baseline(sc, descs, target_paths, S=None):
    """The oracle (tests/ infrastructure, untuned) on a bounded sample of the same workload."""
    import oracle
    S = S or oracle.Scene(sc)
    threads = oracle.default_threads()
    rng = np.random.default_rng(1234)
    per = max(1, target_paths // len(descs))
    nrays, t0 = 0, time.perf_counter()
    for d in descs:
        probes = rng.integers(0, d["width"] * d["height"], per).astype(np.int32)
        _, nr = S.render_probes(d, probes, 0, 1, nthreads=threads)
        nrays += int(nr.sum())
    dt = time.perf_counter() - t0
    return {"value": nrays / dt / 1e6, "unit": "Mrays/s", "cores": threads, "kind": "oracle", "rays": nrays,
            "seconds": dt, "sample": f"{per * len(descs)} paths ({per} random pixels x {len(descs)} frames x 1 spp), "
                                     f"{nrays} rays in {dt:.2f} s wall on {threads} threads"}


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    sc, descs, name = workload(args.config)
    S = oracle.Scene(sc)
    paths = ORACLE_PATHS[args.config]
    for _ in range(args.warmup):
        cpu_baseline(sc, descs, max(len(descs), paths // 4), S)
    rays_total, t_total = 0, 0.0
    cb = None
    for _ in range(args.steps):
        cb = cpu_baseline(sc, descs, paths, S)
        rays_total += cb.pop("rays")
        t_total += cb.pop("seconds")
    value = rays_total / t_total / 1e6  # rays of all K steps / their summed wall time
    cb["value"] = value
    line = {"impl": "reference", "metric": "Mrays/s (transmittance + scattering)", "value": value,
            "unit": "Mrays/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.config == 5 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, paper_2602_05081_b200/inputs.py)",
            "config": {"workload": name + " -- bounded oracle sample per step",
                       "paths_per_step": max(1, paths // len(descs)) * len(descs)},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gabor", choices=["gabor", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--shard", choices=["tiles", "samples"], default=None,
                    help="N > 1 work split: 32x32 tiles (default for config 5, strong scaling) or samples "
                         "(each rank renders its own sample of every frame, weak scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--estimator", default="analytic", choices=["analytic", "tracking", "uniform"],
                    help="scatter estimator: closed-form tau + root (default), delta/ratio tracking, or the "
                         "paper's biased uniform-in-segment free flight (reading U1)")
    ap.add_argument("--foveation", action="store_true",
                    help="foveated rendering variant: gaze at the image centre, all levels in the fovea, "
                         "threshold falling linearly to 0 at eccentricity 0.7 (jitter 0.2)")
    ap.add_argument("--motion-blur", choices=["reference", "culled"], default=None,
                    help="motion-blur variant (direction (1, 0.2, 0), magnitude 0.02): time-sampled reference, "
                         "or the group-culled approximation (attenuation threshold 0.6)")
    ap.add_argument("--adaptive-extent", type=float, default=None, metavar="EPS",
                    help="adaptive clamping variant (Eq. 15): per-primitive extents for threshold EPS")
    ap.add_argument("--tomography", action="store_true",
                    help="tomography variant: the config's scene and views, primary-ray transmittance only (mode 0)")
    ap.add_argument("--streams", type=int, default=2,
                    help="render the frames of a step on this many CUDA streams, each with its own scratch "
                         "(default 2: two frames in flight fill each other's kernel tails)")
    ap.add_argument("--profile-pass", action="store_true", help="only run warmup+steps (for ncu launch lists)")
    args = ap.parse_args()
    rank, local, world = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2602_05081_b200 import gf

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc, descs, name = workload(args.config)
    # the per-view light / camera BVHs live in the scratch buffers the steps share (gf_render
    # reuse_accel): built in the first warm-up render, like the scene BVH; e2e rebuilds everything
    descs = [dict(d, reuse_accel=1) for d in descs]
    if args.tomography:
        descs = [dict(d, mode=0, max_depth=1) for d in descs]
        name += " [tomography: primary-ray transmittance only]"
    if args.estimator == "tracking":
        descs = [dict(d, estimator=1) for d in descs]
        name += " [delta/ratio tracking estimator]"
    if args.estimator == "uniform":
        descs = [dict(d, estimator=2) for d in descs]
        name += " [biased uniform-in-segment free flight (U1)]"
    if args.motion_blur:
        if args.motion_blur == "reference":
            descs = [dict(d, motion_blur=I.motion_blur((1.0, 0.2, 0.0), 0.02)) for d in descs]
        name += f" [motion blur {args.motion_blur}: direction (1, 0.2, 0), magnitude 0.02]"
    f = gf.GaborField(local)
    if args.adaptive_extent:  # adaptive clamping (Eq. 15, C8'): the library's extents, then reload
        f.load_primitives(sc)
        sc = dict(sc, extent=f.adaptive_extent(sc, args.adaptive_extent).cpu().numpy())
        name += f" [adaptive extents, eps {args.adaptive_extent:g}: mean E {float(np.mean(sc['extent'])):.2f}]"
    # BVH keys: (band, level) subtrees (the paper's per-level structures) unless a policy samples orientation
    # bins (Table B2), which then prune per-bin subtrees
    orient = any((d.get(k) or {}).get("orient_strategy", 0) for d in descs for k in ("ext", "nee"))
    bvh_keys = gf.BVH_KEYS_GROUP if orient else gf.BVH_KEYS_LEVEL
    f.set_bvh_keys(bvh_keys)
    torch.cuda.synchronize()
    tb0 = time.perf_counter()
    f.load_primitives(sc)
    f.build_bvh()
    build_s = time.perf_counter() - tb0
    info = f.scene_info()
    if args.motion_blur == "culled":  # the library's group culling (M3) -> a static mask
        mask, _ = f.motion_blur_mask((1.0, 0.2, 0.0), 0.02, 0.6)
        descs = [dict(d, ext=I.policy(static_mask=d["ext"]["static_mask"] & mask),
                      nee=I.policy(static_mask=d["nee"]["static_mask"] & mask)) for d in descs]
    if args.foveation:
        f0 = float(info["level_fmax"].max()) * 1.05
        descs = [dict(d, foveation=I.foveation((d["width"] / 2, d["height"] / 2), f0, f0 / 0.7, 0.2))
                 for d in descs]
        name += " [foveated: gaze centre, threshold 1.05 max level frequency, zero at eccentricity 0.7]"
    # replica check: every rank built the same BVH
    replica = {"bvh_hash": f"{info['bvh_hash']:016x}"}
    shard_kind = args.shard or ("tiles" if args.config == 5 else "samples")
    if world > 1:
        replica["equal_on_all_ranks"] = replica_check(info["bvh_hash"], dist, f.device)
        assert replica["equal_on_all_ranks"], "BVH replicas differ across ranks"
    tiles = shard_kind == "tiles"
    shard = (gf.SHARD_TILES if tiles else gf.SHARD_SAMPLES, rank, world) if world > 1 else (gf.SHARD_NONE, 0, 1)
    spp = 1 if (tiles or world == 1) else world
    H, W = descs[0]["height"], descs[0]["width"]
    nstr = max(1, min(args.streams, len(descs)))
    scratches = [f.render_scratch(descs[0], spp, shard) for _ in range(nstr)]
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(nstr - 1)]
    accum = torch.zeros((len(descs), H * W * 2), dtype=torch.float32, device=f.device)
    rays = torch.zeros(3, dtype=torch.int64, device=f.device)  # camera, extension, NEE
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f.device)  # 256 MB > 126 MB L2

    def step(k, ns=nstr, g=f):
        accum.zero_()
        main = streams[0]
        for s_ in streams[1:ns]:
            s_.wait_stream(main)
        for i, d in enumerate(descs):
            with torch.cuda.stream(streams[i % ns]):
                g.render(d, spp_begin=k * spp, spp_count=spp, shard=shard, accum=accum[i], ray_counts=rays,
                         scratch=scratches[i % ns])
        for s_ in streams[1:ns]:
            main.wait_stream(s_)
        if world > 1:  # tiles: disjoint pixels, gather the image on rank 0; samples: sum of samples
            if tiles:
                dist.reduce(accum, dst=0)
            else:
                dist.all_reduce(accum)

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    if args.profile_pass:
        for k in range(args.steps):
            step(args.warmup + k)
        torch.cuda.synchronize()
        return
    f.stats(reset=True)
    f.set_profiling(timing=True)
    rays.zero_()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed steps, outside the events
            evs[k][0].record()
            step(args.warmup + k)
            evs[k][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    st = f.stats(reset=True)
    f.set_profiling()
    kinds = [int(x) for x in rays.cpu().tolist()]  # camera, extension, NEE (before any further pass)
    psteps = min(args.steps, 2)
    if nstr > 1:  # per-kernel CUDA-event times for the roofline from a one-stream pass (streams overlap)
        f.set_profiling(timing=True)
        for k in range(psteps):
            step(args.warmup + k, 1)
        torch.cuda.synchronize()
        st_stage = f.stats(reset=True)
        f.set_profiling()
        stage_steps = psteps
    else:
        st_stage, stage_steps = st, args.steps
    tt = torch.tensor([t_ms] + [float(x) for x in kinds], dtype=torch.float64, device=f.device)
    if world > 1:
        per_rank = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(per_rank, tt)
        rank_ms = [float(x[0]) / args.steps for x in per_rank]
        t_ms_max = max(float(x[0]) for x in per_rank)
        kinds = [sum(float(x[1 + j]) for x in per_rank) for j in range(3)]
    else:
        rank_ms = [t_ms / args.steps]
        t_ms_max = t_ms
    total_rays = float(sum(kinds))
    value = total_rays / (t_ms_max * 1e-3) / 1e6
    by_kind = {k: v / (t_ms_max * 1e-3) / 1e6 for k, v in zip(("camera", "extension", "nee"), kinds)}

    # ---- counting pass (untimed, one step): algorithmic work per stage
    f.set_profiling(work=True)
    step(args.warmup, 1)
    torch.cuda.synchronize()
    sw = f.stats(reset=True)
    f.set_profiling()
    stage_ms = {k: v for k, v in st_stage["stage_ms"].items() if v > 0}
    dom = max(stage_ms, key=stage_ms.get)
    launches = st_stage["stage_launches"][dom]
    avg_ms = stage_ms[dom] / max(1, launches)
    w = sw["work"][dom]
    nl = max(1, sw["stage_launches"][dom])
    per_launch_bytes = (BYTES_RAY * w["paths"] + BYTES_NODE * w["nodes"] + BYTES_TEST * w["tests"]) / nl
    per_launch_flop = (FLOP_NODE * w["nodes"] + FLOP_TEST * w["tests"] + FLOP_HIT * w["hits"]
                       + FLOP_ERF * w["erf_complex"] + FLOP_ERF_REAL * w["erf_real"]
                       + FLOP_ROOT_EVAL * w["root_evals"]) / nl
    peaks = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6553.0))
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    props = torch.cuda.get_device_properties(local)
    alu_peak = props.multi_processor_count * 128 * 2 * sm_mhz * 1e6 / 1e12
    clocks = clk.summary()
    tr_kernel, traffic, tr_src = load_traffic(args.config, dom)
    kernel = tr_kernel or {"ffA": "k_ffa_pkt (camera rays) / k_ffa_w (extension rays)", "ffB": "k_ffb_w",
                           "nee": "k_nee_w", "tomo": "k_tomo_pkt / k_tomo_w"}.get(dom, dom)
    achieved_gbs = per_launch_bytes / (avg_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": kernel, "stage": dom, "achieved": achieved_gbs, "peak": hbm_peak,
                "unit": "GB/s", "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_ms,
                "bytes_model": f"{BYTES_RAY} B per ray + {BYTES_NODE} B per node box test + {BYTES_TEST} B per "
                               "primitive record tested (SURVEY §8(d) B_ray, uncached), x the work counters of one "
                               "counted step / launches",
                "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                "traffic_source": tr_src,
                "peak_source": "hbm_gbs of MEASURED_PEAKS.json (measured copy bandwidth)",
                "stage_share": {k: v / sum(stage_ms.values()) for k, v in stage_ms.items()},
                "work_per_launch": {k: v / nl for k, v in w.items()}}
    ach_tf = per_launch_flop / (avg_ms * 1e-3) / 1e12
    roofline_alu = {"bound": "alu", "achieved": ach_tf, "peak": alu_peak, "unit": "TFLOP/s", "frac": ach_tf / alu_peak,
                    "peak_source": f"{props.multi_processor_count} SMs x 128 FP32 lanes x 2 FLOP x {sm_mhz:.0f} MHz "
                                   "(sm_max_mhz of MEASURED_PEAKS.json)"}

    # ---- end to end through the public API with host buffers (rank-local, then max over ranks)
    e2e = None
    if not args.no_e2e:
        keys = [k for k in ("mu", "quat", "scale", "alpha", "omega", "extent", "level", "bin", "band") if k in sc]
        host = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).pin_memory() for k in keys}
        out_host = torch.empty_like(accum, device="cpu").pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in host.values())
        d2h = out_host.numel() * out_host.element_size()
        e2e_ms, e2e_rays, e2e_steps = 0.0, 0, []
        g2 = gf.GaborField(local)
        g2.set_bvh_keys(bvh_keys)
        e2e_warm, e2e_n = 1, min(args.steps, 3)
        for k in range(e2e_warm + e2e_n):
            torch.cuda.synchronize()
            rays.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dev = {kk: v.to(f.device, non_blocking=True) for kk, v in host.items()}
            g2.load_primitives(dict(sc, **dev))
            g2.build_bvh()
            step(k, nstr, g2)
            if rank == 0 or not tiles:
                out_host.copy_(accum, non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            if k >= e2e_warm:
                e2e_ms += a.elapsed_time(b)
                e2e_rays += int(rays.sum().item())
                e2e_steps.append(round(a.elapsed_time(b), 3))
        te = torch.tensor([e2e_ms, float(e2e_rays)], dtype=torch.float64, device=f.device)
        if world > 1:
            tm = te.clone()
            dist.all_reduce(tm[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(te[1:], op=dist.ReduceOp.SUM)
            e2e_ms, e2e_rays = float(tm[0]), float(te[1])
        e2e = {"value": e2e_rays / (e2e_ms * 1e-3) / 1e6, "unit": "Mrays/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e2e_n, "ms_per_step": e2e_steps,
               "includes": "pinned H2D of the scene, gf_load_primitives, gf_build_bvh (+ the light and camera BVHs "
                           f"in the first render), gf_render x {len(descs)} frames, D2H of the accumulators"}

    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(sc, descs, ORACLE_PATHS[args.config])
            cb.pop("rays"), cb.pop("seconds")
        line = {"metric": "Mrays/s (transmittance + scattering)", "value": value, "unit": "Mrays/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong" if (tiles and world > 1) or args.config == 5 else "weak",
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded generators, paper_2602_05081_b200/inputs.py; no paper assets)",
                "config": {"workload": name, "config_id": args.config, "n_prims": int(sc["n"]), "image": [W, H],
                           "bvh_keys": "group" if bvh_keys == gf.BVH_KEYS_GROUP else "level",
                           "frames_per_step": len(descs),
                           "frame_masks": [f"{d['ext']['static_mask']:#010x}" for d in descs],
                           "paths_per_step": len(descs) * W * H * (spp if not tiles else 1),
                           "rays_per_step": total_rays / args.steps,
                           "l2": "flushed between timed steps (256 MB write, outside the step events)",
                           "streams": nstr,
                           "accel": "scene BVH built before the timed steps (build_s); the per-view light and camera "
                                    "BVHs built by the first warm-up render and reused (reuse_accel); e2e rebuilds "
                                    "all each step",
                           "build_s": build_s,
                           "parallelism": (f"dp{world} ({shard_kind}-sharded, scene replicated, NCCL "
                                           f"{'reduce of the disjoint tiles' if tiles else 'all-reduce of the samples'} "
                                           "per frame)") if world > 1 else "dp1"},
                "mrays_by_kind": by_kind, "rank_ms_per_step": rank_ms, "replica_check": replica,
                "roofline": roofline, "roofline_alu": roofline_alu, "cpu_baseline": cb, "e2e": e2e,
                "gpu_launches": int(st["launches"]), "clocks": clocks,
                "stage_ms_per_step": {k: v / stage_steps for k, v in stage_ms.items()},
                "work_per_step": {k: {kk: vv for kk, vv in v.items() if vv}
                                  for k, v in sw["work"].items() if any(v.values())}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
