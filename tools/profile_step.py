"""Small fixed-count run of the headline config for profiling (ncu launch
lists / full captures): W warm-up + K timed MM iterations, no CPU baseline."""
import argparse
import sys

sys.path.insert(0, ".")
from paper_2206_03410_b200 import registration as R  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--max-ctas", type=int, default=0)
ap.add_argument("--no-timing", action="store_true")
a = ap.parse_args()
p = R.make_problem(a.config, scale=a.scale)
ctx = R.Context(max_ctas=a.max_ctas)
ctx.set_problem(p)
prm = ctx.init_parameters()
cfg = R.solver_config(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300,
                      i_max=a.warmup + a.iters + 5)
ctx.enable_timing(not a.no_timing)
ctx.begin(cfg)
ctx.iterate(a.warmup)
s0 = ctx.stats()
acc, done, ms = ctx.iterate(a.iters)
s1 = ctx.stats()
ctx.finish()
print("iters", acc, "device ms/iter", ms / acc, "pcg iters/iter", (s1["pcg_iterations"] - s0["pcg_iterations"]) / acc)
print({k: (s1["kernel_ms"][k] - s0["kernel_ms"][k]) / acc for k in s1["kernel_ms"]})
