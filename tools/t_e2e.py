"""Timing breakdown of one bench e2e step (diagnostic)."""
import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2602_05081_b200 import gf, inputs as I
sc = I.scene_cfg2()
f = gf.GaborField(0)
f.load_primitives(sc); f.build_bvh()
descs = [dict(I.render_desc_cfg2(i), reuse_accel=1) for i in range(4)]
scratch = f.render_scratch(descs[0], 1)
accum = torch.zeros((4, 1024 * 1024 * 2), device='cuda')
rays = torch.zeros(3, dtype=torch.int64, device='cuda')
keys = ("mu", "quat", "scale", "alpha", "omega", "extent", "level", "bin")
host = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).pin_memory() for k in keys}
out_host = torch.empty_like(accum, device="cpu").pin_memory()
g2 = gf.GaborField(0)
def tm(label, fn):
    torch.cuda.synchronize(); a = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{label:28s} {(time.perf_counter() - a) * 1e3:8.2f} ms"); return r
for step in range(3):
    print("step", step)
    dev = tm("h2d", lambda: {kk: v.to('cuda', non_blocking=True) for kk, v in host.items()})
    tm("load", lambda: g2.load_primitives(dict(sc, **dev)))
    tm("build", lambda: g2.build_bvh())
    for i, d in enumerate(descs):
        tm(f"render {i}", lambda: g2.render(d, 0, 1, accum=accum[i], ray_counts=rays, scratch=scratch))
    tm("d2h", lambda: out_host.copy_(accum, non_blocking=True))
