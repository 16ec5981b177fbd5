"""diagnostic: per-sample disagreement of the cfg2 full-frame render with the oracle (GF_LIB selects the lib)."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2602_05081_b200 import gf, inputs as I
sc = I.scene_cfg2()
f = gf.GaborField(0); f.load_primitives(sc); f.build_bvh()
S = oracle.Scene(sc)
rng = np.random.default_rng(7)
for mi in (1, 3):
    d = I.render_desc_cfg2(mi)
    acc, _ = f.render(d)
    acc = acc.view(-1, 2).cpu().numpy()[:, 0].astype(np.float64)
    pix = rng.integers(0, 1024 * 1024, 600)
    vo, _ = S.render_probes(d, pix, 0, 1)
    vg = acc[pix]
    rel = np.abs(vg - vo[:, 0]) / (np.abs(vo[:, 0]) + 1e-2)
    print(os.environ.get("GF_LIB", "default").split("/")[-1], "mask", mi, "flips>1e-3: %.4f  >1e-2: %.4f  mean gpu %.5f oracle %.5f" % ((rel > 1e-3).mean(), (rel > 1e-2).mean(), vg.mean(), vo[:, 0].mean()))
