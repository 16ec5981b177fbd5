"""Bias of the GF_EST_UNIFORM free flight (reading U1: t* uniform in the crossing bin
instead of the root) against the exact analytic estimator, measured on the GPU on the same Philox
streams: config 2 (single scattering, 512^2, mask {0..3}) and config 3 (clouds, depth 8, 256^2),
64 spp each, and config 5 (army, depth 8, 512^2, full mask, 16 spp).  Reports the image-mean relative bias, the mean |per-pixel bias| in units of its
standard error, and the stage times of both estimators.  Output: one JSON object on stdout."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05081_b200 import gf, inputs as I  # noqa: E402


def run(sc, desc, spp):
    f = gf.GaborField(0)
    f.load_primitives(sc)
    f.build_bvh()
    out = {}
    for name, est in (("analytic", 0), ("uniform", 2)):
        f.set_profiling(timing=True)
        acc, _ = f.render(dict(desc, estimator=est), 0, spp)
        torch.cuda.synchronize()
        st = f.stats(reset=True)
        f.set_profiling()
        a = acc.view(-1, 2).double().cpu().numpy()
        mean = a[:, 0] / spp
        var = np.maximum(a[:, 1] / spp - mean ** 2, 0.0) / spp
        out[name] = (mean, var, {k: round(v, 2) for k, v in st["stage_ms"].items() if v > 0})
    ma, va, ta = out["analytic"]
    mu, vu, tu = out["uniform"]
    se = np.sqrt(va + vu)
    z = np.abs(mu - ma)[se > 0] / se[se > 0]
    return {"image_mean_analytic": float(ma.mean()), "image_mean_uniform": float(mu.mean()),
            "relative_bias": float((mu.mean() - ma.mean()) / ma.mean()),
            "mean_abs_z_per_pixel": float(z.mean()), "frac_pixels_z_gt_3": float((z > 3).mean()),
            "stage_ms_analytic": ta, "stage_ms_uniform": tu}


res = {"cfg2": run(I.scene_cfg2(), I.render_desc_cfg2(3, 512, 512), 64),
       "cfg3": run(I.scene_cfg3(), I.render_desc_cfg3(256, 256), 64),
       "cfg5": run(I.scene_cfg5(), I.render_desc_cfg5((0, 1, 2, 3), 512, 512), 16)}
print(json.dumps(res))
