"""Wall-clock breakdown of the one-shot register path's host setup (config 2)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2206_03410_b200 import registration as R  # noqa: E402

p = R.make_problem(2)
ctx = R.Context()
for rep in range(3):
    t0 = time.perf_counter()
    ctx.set_target(p.target)
    t1 = time.perf_counter()
    ctx.set_problem(p)
    t2 = time.perf_counter()
    prm = ctx.init_parameters()
    t3 = time.perf_counter()
    cfg = R.solver_config(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300, i_max=30)
    X, v, rep_ = ctx.register(cfg, one_shot_problem=p)
    t4 = time.perf_counter()
    print(f"set_target {1e3*(t1-t0):.1f} ms, set_problem {1e3*(t2-t1):.1f} ms, init_parameters {1e3*(t3-t2):.1f} ms, "
          f"one-shot register (30 it) {1e3*(t4-t3):.1f} ms")
