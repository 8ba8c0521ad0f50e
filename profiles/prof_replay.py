import cProfile
import pstats
import sys

sys.path.insert(0, ".")
sys.argv = ["x"]
import runpy  # noqa: E402

g = runpy.run_path("profiles/one_replay.py")
once = g["once"]
pr = cProfile.Profile()
pr.enable()
for k in range(10):
    once(100 + k)
import torch  # noqa: E402

torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
