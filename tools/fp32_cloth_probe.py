"""fp32 vs f64 cloth sheet (33 x 33 on the configs[2] sphere): per-step sphere
impulse (z) and position drift, for choosing the test's window and bounds."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2503_05046_b200 as mp  # noqa: E402
from paper_2503_05046_b200 import scenes  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
sc = scenes.cloth_sheet_scene(n_side=33)
sc["cloth"][0]["center"][2] = 0.26
sc["solver"]["eps_r"] = 1e-4
st = {k: scenes.build_state(sc, precision=p) for k, p in (("a", "f64"), ("a2", "f64"), ("b", "f32"))}
series = {k: [] for k in st}
dx, dx2 = [], []
for i in range(steps):
    for k, s in st.items():
        series[k].append(float(mp.advance_step(s).wrench[0][2]))
    xa = st["a"].particles.x.cpu().numpy()
    dx.append(float(np.abs(xa - st["b"].particles.x.cpu().numpy()).max()) / sc["h"])
    dx2.append(float(np.abs(xa - st["a2"].particles.x.cpu().numpy()).max()) / sc["h"])
cum = {k: np.cumsum(v) for k, v in series.items()}
print(json.dumps(dict(steps=steps, dx_over_h=dx[-1], dx_max=max(dx),
                      dx_f64_repeat_over_h=dx2[-1], dx_f64_repeat_max=max(dx2),
                      z_series={k: [round(x, 4) for x in v] for k, v in series.items()},
                      cum_rel_f32=float(abs(cum["b"][-1] - cum["a"][-1]) / abs(cum["a"][-1])),
                      cum_rel_f64_repeat=float(abs(cum["a2"][-1] - cum["a"][-1]) / abs(cum["a"][-1])))))
