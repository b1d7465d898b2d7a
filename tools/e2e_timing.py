"""Where the one-shot (fresh context) e2e time goes on config 2."""
import sys
import time

sys.path.insert(0, ".")
from paper_2206_03410_b200 import registration as R  # noqa: E402

p = R.make_problem(2)
warm = R.Context()
prm = None
warm.set_problem(p)
prm = warm.init_parameters()
cfg = R.solver_config(nu_a_init=prm["nu_a"], nu_a_min=prm["nu_a"], nu_r_init=prm["nu_r"], eps=1e-300, i_max=30)
warm.register(cfg, one_shot_problem=p)
for rep in range(3):
    t0 = time.perf_counter()
    c = R.Context()
    t1 = time.perf_counter()
    c.register(cfg, one_shot_problem=p)
    t2 = time.perf_counter()
    c.register(cfg, one_shot_problem=p)
    t3 = time.perf_counter()
    c.close()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms, first register {1e3*(t2-t1):.1f} ms, second register {1e3*(t3-t2):.1f} ms, "
          f"close {1e3*(t4-t3):.1f} ms")
