"""Standalone check of the fused TMA chain: bitwise equality with the unfused
path (RK_NO_CHAIN) and timing, via rk_precond_apply (5+1 sweeps)."""
import os, subprocess, sys, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def run(n, radius):
    import paper_1501_03358_b200 as rk
    from problems.stencils import porous7
    prob = porous7(n, radius)
    ctx = rk.Context(0)
    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets,
                         torch.from_numpy(prob.bands()).cuda(), prob.periodic)
    r = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, prob.N)).cuda()
    z = op.precond(r)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        op.precond(r, z)
    ev0.record(); K = 20
    for _ in range(K):
        op.precond(r, z)
    ev1.record(); torch.cuda.synchronize()
    return z.cpu().numpy(), ev0.elapsed_time(ev1) / K

if __name__ == "__main__":
    if len(sys.argv) > 1:
        z, ms = run(int(sys.argv[1]), int(sys.argv[2]))
        np.save(sys.argv[3], z); print(json.dumps({"ms": ms}))
        sys.exit(0)
    for n, rad in ((64, 4), (128, 6)):
        out = {}
        for mode in ("chain", "nochain"):
            env = dict(os.environ)
            if mode == "nochain": env["RK_NO_CHAIN"] = "1"
            p = subprocess.run([sys.executable, __file__, str(n), str(rad), f"/tmp/z_{mode}.npy"],
                               env=env, capture_output=True, text=True, timeout=120)
            print(mode, p.stdout.strip(), p.stderr[-500:])
            out[mode] = (np.load(f"/tmp/z_{mode}.npy"), json.loads(p.stdout.strip().splitlines()[-1])["ms"])
        a, b = out["chain"][0], out["nochain"][0]
        print(f"n={n}: bitwise_equal={np.array_equal(a, b)} maxdiff={np.max(np.abs(a-b)):.3e} "
              f"chain {out['chain'][1]*1e3:.1f} us  unfused {out['nochain'][1]*1e3:.1f} us per M^-1")
