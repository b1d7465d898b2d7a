"""Sweep PCG tolerance / coarse aggregation on the headline config: ms per solve, iterations."""
import os
import subprocess
import sys

sys.path.insert(0, ".")
for env in ["NRR_AGG_CTAS=4", "NRR_AGG_CTAS=6", "NRR_AGG_CTAS=8"]:
    for rtol in ["1e-10"]:
        code = ("import sys; sys.path.insert(0,'.'); from paper_2206_03410_b200 import registration as R\n"
                "p=R.make_problem(2); ctx=R.Context(pcg_rtol=%s); ctx.set_problem(p); prm=ctx.init_parameters()\n"
                "cfg=R.solver_config(nu_a_init=prm['nu_a'],nu_a_min=prm['nu_a'],nu_r_init=prm['nu_r'],eps=1e-300,i_max=20)\n"
                "ctx.enable_timing(True); ctx.begin(cfg); ctx.iterate(3); s0=ctx.stats(); a,d,ms=ctx.iterate(8); s1=ctx.stats()\n"
                "print('%s rtol %s: step ms %%.3f pcg ms %%.3f pcg its %%.1f' %% (ms/8, (s1['kernel_ms']['pcg']-s0['kernel_ms']['pcg'])/8, (s1['pcg_iterations']-s0['pcg_iterations'])/8))"
                % (rtol, env, rtol))
        e = dict(os.environ)
        k, v = env.split("=")
        e[k] = v
        r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-300:], flush=True)
