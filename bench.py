#!/usr/bin/env python
"""Benchmark: Mrays/s (transmittance + scattering) of the Gabor Fields hot path on B200.

Workload (BASELINE.json configs[1], "config 2"): bunny-like 100k-primitive Gabor field,
1024x1024, single scattering, 4 static LOD levels ({0}, {0,1}, {0..2}, {0..3}), 1 spp per
level per GPU.  One step = one frame per LOD level = 4 x 1024^2 paths through gf_render
(free flight + NEE); with N GPUs each rank renders its own sample of every frame
(sample-sharded, scene replicated, weak scaling) and the frame accumulators are summed with
one NCCL all-reduce per step (the only exchange).  A "ray" is one ray query: camera,
extension (free-flight) or NEE shadow ray.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config 1|2]
"""
import argparse
import json
import math
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
# FP32 algorithmic work model per unit: node slab test, primitive whitening test,
# hit setup, and one complex-erf endpoint (Horner, kErfTerms complex terms, 4 FFMA = 8 FLOP each).
ERF_TERMS = 30
FLOP_NODE, FLOP_TEST, FLOP_HIT, FLOP_ERF = 24, 45, 40, 8 * ERF_TERMS
FLOP_ERF_REAL = 20  # real erf (Omega = 0): erff, ~10 FFMA
FLOP_ROOT_EVAL = 20  # per root-finder evaluation (kappa term, excluding its erf endpoints)


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


def load_traffic(config, stage):
    """(kernel, DRAM bytes per launch) of the stage's kernel from the committed ncu --set full
    capture, or (None, None)."""
    try:
        t = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")))
        e = t[f"cfg{config}"][stage]
        return e["kernel"], e["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None, None


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
    elif config == 3:
        sc = I.scene_cfg3()
        descs = [I.render_desc_cfg3()]
        name = ("cfg3: procedural clouds, 327,600 primitives (15,600 Gaussian cores + 312,000 Gabors), 1024x1024, "
                "multiple scattering depth 8, full LOD, 1 spp per step per GPU")
    elif config == 4:
        sc = I.scene_cfg4()
        descs = [I.render_desc_cfg4()]
        name = ("cfg4: dense 1M-primitive asset, 2048x2048, multiple scattering depth 8, stochastic per-recursion "
                "masks (PL+CV Accum. beta 0.2 x orientation Importance, Zero NEE), 1 spp per step per GPU")
    elif config == 5:
        sc = I.scene_cfg5()
        descs = [I.render_desc_cfg5(lv, 4096, 4096) for lv in ((0,), (0, 1), (0, 1, 2), (0, 1, 2, 3))]
        name = ("cfg5: 4M-primitive army (120 x 33,280-primitive bunnies), 4096x4096, multiple scattering depth 8, "
                "LOD sweep over 4 global static masks, 1 spp per mask per step per GPU")
    else:
        sc = I.scene_cfg2()
        descs = [I.render_desc_cfg2(i) for i in range(4)]
        name = ("cfg2: bunny-like 100k-primitive Gabor field, 1024x1024, single scattering, 4 static LOD levels "
                "({0},{0,1},{0..2},{0..3}), 1 spp per level per GPU")
    return sc, descs, name


# ----------------------------------------------------------------------------------------------
def cpu_baseline(sc, descs, target_paths):
    """The oracle (tests/ infrastructure, untuned) on a bounded sample of the same workload."""
    import oracle
    S = oracle.Scene(sc)
    threads = oracle.default_threads()
    rng = np.random.default_rng(1234)
    per = max(1, target_paths // len(descs))
    nrays, t0 = 0, time.perf_counter()
    for d in descs:
        probes = rng.integers(0, d["width"] * d["height"], per).astype(np.int32)
        _, nr = S.render_probes(d, probes, 0, 1, nthreads=threads)
        nrays += int(nr.sum())
    dt = time.perf_counter() - t0
    return {"value": nrays / dt / 1e6, "unit": "Mrays/s", "cores": threads, "kind": "oracle", "rays": nrays, "seconds": dt,
            "sample": f"{per * len(descs)} paths ({per} probe pixels x {len(descs)} LOD levels x 1 spp), "
                      f"{nrays} rays in {dt:.2f} s wall on {threads} threads"}


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    sc, descs, name = workload(args.config)
    paths = 1024
    for _ in range(args.warmup):
        cpu_baseline(sc, descs, paths // 4)
    rays_total, t_total = 0, 0.0
    cb = None
    for _ in range(args.steps):
        cb = cpu_baseline(sc, descs, paths)
        rays_total += cb.pop("rays")
        t_total += cb.pop("seconds")
    value = rays_total / t_total / 1e6  # rays of all K steps / their summed wall time
    cb["value"] = value
    line = {"impl": "reference", "metric": "Mrays/s (transmittance + scattering)", "value": value,
            "unit": "Mrays/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded generators, paper_2602_05081_b200/inputs.py)",
            "config": {"workload": name + " -- bounded oracle sample per step", "paths_per_step": paths},
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
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--estimator", default="analytic", choices=["analytic", "tracking"],
                    help="scatter estimator: closed-form tau + root (default) or delta/ratio tracking")
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
                    help="render the LOD frames of a step on this many CUDA streams, each with its own scratch "
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
    # the per-view light / camera BVHs live in the one scratch buffer the steps share (gf_render
    # reuse_accel): built in the first warm-up render, like the scene BVH; e2e rebuilds everything
    descs = [dict(d, reuse_accel=1) for d in descs]
    if args.tomography:
        descs = [dict(d, mode=0, max_depth=1) for d in descs]
        name += " [tomography: primary-ray transmittance only]"
    if args.estimator == "tracking":
        descs = [dict(d, estimator=1) for d in descs]
        name += " [delta/ratio tracking estimator]"
    if args.adaptive_extent:
        sc = dict(sc, extent=I.adaptive_extent(sc, args.adaptive_extent))
        name += f" [adaptive extents, eps {args.adaptive_extent:g}: mean E {float(np.mean(sc['extent'])):.2f}]"
    if args.motion_blur:
        mdir, mm = (1.0, 0.2, 0.0), 0.02
        if args.motion_blur == "reference":
            descs = [dict(d, motion_blur=I.motion_blur(mdir, mm)) for d in descs]
        else:
            mask, _ = I.motion_blur_mask(sc, mdir, mm, 0.6)
            descs = [dict(d, ext=I.policy(static_mask=d["ext"]["static_mask"] & mask),
                          nee=I.policy(static_mask=d["nee"]["static_mask"] & mask)) for d in descs]
        name += f" [motion blur {args.motion_blur}: direction (1, 0.2, 0), magnitude 0.02]"
    if args.foveation:
        lf = I.level_fmax(sc)
        f0 = float(lf.max()) * 1.05
        descs = [dict(d, foveation=I.foveation(sc, (d["width"] / 2, d["height"] / 2), f0, f0 / 0.7, 0.2))
                 for d in descs]
        name += " [foveated: gaze centre, threshold 1.05 max level frequency, zero at eccentricity 0.7]"
    f = gf.GaborField(local)
    f.load_primitives(sc, group_f0=I.group_f0(sc))
    f.build_bvh()
    H, W = descs[0]["height"], descs[0]["width"]
    shard = (gf.SHARD_SAMPLES, rank, world)
    scratch = f.render_scratch(descs[0], 1, shard)
    nstr = max(1, min(args.streams, len(descs)))
    scratches = [scratch] + [f.render_scratch(descs[0], 1, shard) for _ in range(nstr - 1)]
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(nstr - 1)]
    accum = torch.zeros((len(descs), H * W * 2), dtype=torch.float32, device=f.device)
    rays = torch.zeros(2, dtype=torch.int64, device=f.device)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f.device)  # 256 MB > 126 MB L2

    def step(k, ns=nstr):
        accum.zero_()
        main = streams[0]
        for s_ in streams[1:ns]:
            s_.wait_stream(main)
        for i, d in enumerate(descs):
            with torch.cuda.stream(streams[i % ns]):
                f.render(d, spp_begin=k * world, spp_count=world, shard=shard, accum=accum[i], ray_counts=rays,
                         scratch=scratches[i % ns])
        for s_ in streams[1:ns]:
            main.wait_stream(s_)
        if world > 1:
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
    nrays = int(rays.sum().item())  # (before any further pass adds to the counter)
    if nstr > 1:  # per-kernel CUDA-event times for the roofline from a one-stream pass (streams overlap)
        f.set_profiling(timing=True)
        for k in range(args.steps):
            step(args.warmup + k, 1)
        torch.cuda.synchronize()
        st_stage = f.stats(reset=True)
        f.set_profiling()
    else:
        st_stage = st
    tt = torch.tensor([t_ms, float(nrays)], dtype=torch.float64, device=f.device)
    if world > 1:
        tmax = tt.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        t_ms_max, total_rays = float(tmax[0]), float(tt[1])
    else:
        t_ms_max, total_rays = t_ms, float(nrays)
    value = total_rays / (t_ms_max * 1e-3) / 1e6

    # ---- counting pass (untimed) on the same samples: algorithmic work per stage
    f.set_profiling(work=True)
    for k in range(args.steps):
        step(args.warmup + k)
    torch.cuda.synchronize()
    sw = f.stats(reset=True)
    f.set_profiling()
    stage_ms = {k: v for k, v in st_stage["stage_ms"].items() if v > 0}
    dom = max(stage_ms, key=stage_ms.get)
    launches = st_stage["stage_launches"][dom]
    w = sw["work"][dom]
    flops = (FLOP_NODE * w["nodes"] + FLOP_TEST * w["tests"] + FLOP_HIT * w["hits"] + FLOP_ERF * w["erf_complex"]
             + FLOP_ERF_REAL * w["erf_real"] + FLOP_ROOT_EVAL * w["root_evals"])
    per_launch_flop = flops / max(1, sw["stage_launches"][dom])
    avg_ms = stage_ms[dom] / max(1, launches)
    achieved = per_launch_flop / (avg_ms * 1e-3) / 1e12
    peaks = load_peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    props = torch.cuda.get_device_properties(local)
    peak = props.multi_processor_count * 128 * 2 * sm_mhz * 1e6 / 1e12
    clocks = clk.summary()
    tr_kernel, traffic = load_traffic(args.config, dom)
    kernel = tr_kernel or {"ff": "k_ff_pkt (depth 0, static masks) / k_ff", "nee": "k_nee_w", "tomo": "k_tomo_pkt (static masks) / k_tomo_w",
                           "ff_fallback": "k_ffA+k_ffB"}.get(dom, dom)
    roofline = {"bound": "alu", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                "profiles/r01_traffic.json)",
                "peak_source": f"{props.multi_processor_count} SMs x 128 FP32 lanes x 2 FLOP x {sm_mhz:.0f} MHz "
                               "(sm_max_mhz of MEASURED_PEAKS.json)",
                "stage_share": {k: v / sum(stage_ms.values()) for k, v in stage_ms.items()},
                "work_per_launch": {k: v / max(1, sw["stage_launches"][dom]) for k, v in w.items()}}

    # ---- end to end through the public API with host buffers (rank-local, then max over ranks)
    e2e = None
    if not args.no_e2e:
        keys = ("mu", "quat", "scale", "alpha", "omega", "extent", "level", "bin")
        host = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).pin_memory() for k in keys}
        out_host = torch.empty_like(accum, device="cpu").pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in host.values())
        d2h = out_host.numel() * out_host.element_size()
        e2e_ms, e2e_rays, e2e_steps = 0.0, 0, []
        g2 = gf.GaborField(local)
        e2e_warm = 2
        for k in range(e2e_warm + args.steps):
            torch.cuda.synchronize()
            rays.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dev = {kk: v.to(f.device, non_blocking=True) for kk, v in host.items()}
            scd = dict(sc, **dev)
            g2.load_primitives(scd, group_f0=I.group_f0(sc))
            g2.build_bvh()
            accum.zero_()
            for s_ in streams[1:]:
                s_.wait_stream(streams[0])
            for i, d in enumerate(descs):  # same stream layout as the timed steps
                with torch.cuda.stream(streams[i % nstr]):
                    g2.render(d, spp_begin=k * world, spp_count=world, shard=shard, accum=accum[i],
                              ray_counts=rays, scratch=scratches[i % nstr])
            for s_ in streams[1:]:
                streams[0].wait_stream(s_)
            if world > 1:
                dist.all_reduce(accum)
            out_host.copy_(accum, non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            if k >= e2e_warm:  # the first iterations are warm-up
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
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_steps,
               "includes": "pinned H2D of the scene, gf_load_primitives, gf_build_bvh, gf_render x 4 levels, "
                           "D2H of the accumulators"}

    if rank == 0:
        cb = None
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(sc, descs, {1: 4096, 2: 4096, 3: 512, 4: 32, 5: 16}[args.config])
            cb.pop("rays"), cb.pop("seconds")
        line = {"metric": "Mrays/s (transmittance + scattering)", "value": value, "unit": "Mrays/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded generators, paper_2602_05081_b200/inputs.py; no paper assets)",
                "config": {"workload": name, "n_prims": int(sc["n"]), "image": [W, H], "lod_levels": len(descs),
                           "paths_per_step": len(descs) * W * H * world,
                           "rays_per_step": total_rays / args.steps,
                           "l2": "flushed between timed steps (256 MB write, outside the step events)",
                           "streams": nstr,
                           "accel": "scene BVH built before the timed steps; the per-view light and camera BVHs "
                                    "built by the first warm-up render and reused (reuse_accel); e2e rebuilds all "
                                    "each step",
                           "parallelism": f"dp{world} (sample-sharded, scene replicated, NCCL all-reduce of "
                                          "accumulators per step)" if world > 1 else "dp1"},
                "roofline": roofline, "cpu_baseline": cb, "e2e": e2e,
                "gpu_launches": int(st["launches"]), "clocks": clocks,
                "stage_ms_per_step": {k: v / args.steps for k, v in stage_ms.items()},
                "work_per_step": {k: {kk: vv / args.steps for kk, vv in v.items() if vv}
                                  for k, v in sw["work"].items() if any(v.values())}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
