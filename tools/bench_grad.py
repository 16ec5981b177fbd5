"""Backward throughput (diagnostic, not the bench line): gf_trace_grad_params (+ finish) and
gf_trace_grad_alpha against the forward gf_trace_transmittance on the same rays -- the config-2
scene, one 1024x1024 camera view (pixel centres), each of the 4 static LOD masks; CUDA events on
the launching stream, 3 warm-ups, inputs resident (rays 32 MB; scene + BVH L2-resident)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_05081_b200 import gf, inputs as I  # noqa: E402

sc = I.scene_cfg2()
f = gf.GaborField(0)
f.load_primitives(sc)
f.build_bvh()
d = I.render_desc_cfg2(3)
idx = np.arange(d["width"] * d["height"])
o, v = I.camera_rays_f64(d, idx % d["width"], idx // d["width"])
rays = torch.as_tensor(I.pack_rays(o, v)).cuda()
# the same rays in 8x4 pixel blocks (GF_TRACE_PACKETS wants 32 coherent consecutive rays)
W_, H_ = d["width"], d["height"]
by, bx, ly, lx = np.meshgrid(np.arange(H_ // 4), np.arange(W_ // 8), np.arange(4), np.arange(8), indexing="ij")
blk = ((by * 4 + ly) * W_ + bx * 8 + lx).reshape(-1)
rays_blk = rays[torch.as_tensor(blk).cuda()].contiguous()
n = rays.shape[0]
dl = torch.randn(n, device="cuda")
acc = torch.zeros((f.n, 16), device="cuda")
ga = torch.zeros(f.n, device="cuda")


def timed(fn, reps=5):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {}
for li, lv in enumerate(I.CFG2_LOD_LEVELS):
    f.set_lod_mask({"static_mask": I.level_mask(lv)})
    fwd = timed(lambda: f.trace_transmittance(rays))
    gpar = timed(lambda: f.trace_grad_params(rays, dl, accum=acc))
    gpk = timed(lambda: f.trace_grad_params(rays_blk, dl, accum=acc, packets=True))
    gal = timed(lambda: f.trace_grad_alpha(rays, dl, out=ga))
    out[str(lv)] = {"forward_ms": fwd, "grad_params_ms": gpar, "grad_params_packets_ms": gpk, "grad_alpha_ms": gal,
                    "forward_Mrays_s": n / fwd / 1e3, "grad_params_Mrays_s": n / gpar / 1e3,
                    "grad_params_packets_Mrays_s": n / gpk / 1e3}
print(json.dumps({"rays": n, "scene": "cfg2 (100k primitives)", "per_mask": out}, indent=1))
