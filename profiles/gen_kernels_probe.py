import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json, numpy as np
from paper_1306_3277_b200 import generic, RngStream
from paper_1306_3277_b200.inference import particle_filter, build_filter_grid
FIX=json.load(open(os.path.join(sys.path[0], 'tests/golden/gen_models.json')))
d=dict(FIX["lowered"]["Lorenz96"]); d.pop("fingerprint",None)
m=generic.from_description(d)
g=np.load(os.path.join(sys.path[0], 'tests/golden/pf.npz'))
grid=build_filter_grid(0.0, 2.0, 40, g["l96/obs_t"], g["l96/obs_v"], g["l96/obs_m"], n_obs=8)
out=particle_filter(m, g["l96/theta"], grid, RngStream(1), n_particles=1<<16, exact=False)
print(out.loglik)
