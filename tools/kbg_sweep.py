import sys, torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2012_09499_b200.plan import SrpPlan
scene, pm, pmp, bounds, tdoa, omega = bench.workload(0)
Y = torch.from_numpy(scene.Y).cuda()
for kbg in (4, 8, 32):
    plan = SrpPlan(tdoa, pm, pmp, bounds, omega, sample_period=bench.T, n_aux=4, weights="stored", kb_per_group=kbg)
    psi, _ = plan.cross_spectra(Y)
    xi = plan.lattice(psi)
    for maps in (True, False):
        for _ in range(3): plan.approx(xi, maps=maps)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(10): plan.approx(xi, maps=maps)
        b.record(); b.synchronize()
        print(f"kb_per_group={kbg} maps={maps}: approx (split+K4+idx) {a.elapsed_time(b)/10*1e3:.1f} us")
