#!/usr/bin/env python
"""Time K4/K2 with single-CTA tiles vs CTA pairs (SRPB_TC_PAIR=0/1), separate
processes: python tools/pair_sweep.py"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, torch
sys.path.insert(0, %r)
import bench
from paper_2012_09499_b200.plan import SrpPlan
scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
Y = torch.from_numpy(scene.Y).cuda()
for kbg in (4, 10):
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=4, weights="stored", kb_per_group=kbg)
    psi, _ = plan.cross_spectra(Y); xi = plan.lattice(psi)
    for name, fn in (("approx", lambda: plan.approx(xi)), ("conv", lambda: plan.conventional(psi))):
        if name == "conv" and kbg != 4: continue
        for _ in range(3): fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        n = 10 if name == "approx" else 3
        for _ in range(n): fn()
        b.record(); b.synchronize()
        print(f"  kbg={kbg} {name}: {a.elapsed_time(b)/n*1e3:.1f} us", flush=True)
''' % ROOT
for pair in ("0", "1"):
    env = dict(os.environ, SRPB_TC_PAIR=pair)
    print("pair", pair, flush=True)
    subprocess.run([sys.executable, "-c", CODE], env=env, check=False, timeout=300)
