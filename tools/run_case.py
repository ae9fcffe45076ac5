"""Run the full GPU pipeline once on a (possibly scaled-down) config: python tools/run_case.py CFG [g N R]."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2405_14892_b200 as mvn
cfg = W.CONFIGS[sys.argv[1]]
if len(sys.argv) > 2:
    g, N, R = map(int, sys.argv[2:5])
    cfg = W.small_config(cfg.name + "-small", g, N, R, base=cfg.name)
inp = W.make_inputs(cfg)
t = time.time()
out = mvn.mvn_crd(inp.xy, inp.mu, cfg.sigma2, cfg.beta, cfg.nu, cfg.nugget, cfg.u, cfg.N, cfg.R, cfg.seed_lattice, cfg.conf)
print(cfg.name, "n", cfg.n, "NR", cfg.NR, "info", out.info, "k*", list(out.k_star), "logP[-1]", out.logP[-1], "ms", [round(x, 2) for x in out.ms_stage], "wall", time.time() - t)
