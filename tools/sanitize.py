"""Small driver for compute-sanitizer: exercises every kernel family of libgf.so on
config-1 and a scaled-down config-2 scene (tomography, trace, candidates, single and multiple
scattering with packets / warp free flight / NEE, stochastic masks, tracking estimator, gradients).

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_05081_b200 import gf  # noqa: E402
from paper_2602_05081_b200 import inputs as I  # noqa: E402


def main():
    import torch
    small = "--small" in sys.argv
    # config 1: tomography (warp + forced packets), trace, candidates, gradients
    sc = I.scene_cfg1()
    f = gf.GaborField(0)
    f.load_primitives(sc)
    f.build_bvh()
    d = I.render_desc_cfg1(32, 32)
    f.render(d)
    os.environ["GF_DEBUG_TOMO_PKT_MIN"] = "1"
    f.render(d)
    del os.environ["GF_DEBUG_TOMO_PKT_MIN"]
    rays = I.rays_through_box(7, 256)
    f.trace_transmittance(rays, counters=True)
    f.trace_transmittance(rays, brute_force=True)
    f.trace_candidates(rays, capacity=64)
    f.trace_grad_alpha(rays, np.ones(256, np.float32))
    f.trace_grad_params(rays, np.ones(256, np.float32))
    f.trace_grad_params(rays, np.ones(256, np.float32), packets=True)
    f.set_lod_mask(I.policy(level_strategy=5, beta=0.2, orient_strategy=3))
    f.trace_transmittance(rays, seed=3)
    # scaled-down config 2: single scattering (packets + NEE over the light BVH), multiple
    # scattering with stochastic masks (warp free flight), tracking estimator
    sc2 = I.scene_bunny(counts=(150, 1050, 2800, 6000) if small else (600, 4200, 11200, 24000))
    g = gf.GaborField(0)
    g.load_primitives(sc2)
    g.build_bvh()
    w = 32 if small else 64
    g.render(I.render_desc_cfg2(3, w, w))
    d4 = I.render_desc_cfg4(w, w)
    d4.update(I.camera((0, 0.3, 3.2), (0, 0.05, 0), (0, 1, 0), 40.0, w, w))
    d4["max_depth"] = 3
    g.render(d4)
    d3 = dict(I.render_desc_cfg2(3, w, w), max_depth=3, estimator=1)
    g.render(d3)
    probes = torch.arange(0, w * w, 7, dtype=torch.int32)
    g.render(I.render_desc_cfg2(2, w, w), 0, 2, probes=probes)
    torch.cuda.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
