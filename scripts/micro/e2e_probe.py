"""e2e vs device-buffer solve timing breakdown on c3 (experiment)."""
import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1501_03358_b200 as rk
from problems import get_workload
w = get_workload('c3'); prm = w.params; prob = w.problem()
ctx = rk.Context(0)
op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets, torch.from_numpy(prob.bands()).cuda(), prob.periodic)
s = rk.Solver(op, rk.config_from_params(prm))
T = 20
B = [torch.from_numpy(prob.rhs(t).reshape(-1)).cuda() for t in range(T)]
Bh = [b.cpu().pin_memory() for b in B]
Xh = [torch.zeros(prob.N, dtype=torch.float64).pin_memory() for _ in range(T)]
X = [torch.zeros(prob.N, dtype=torch.float64, device='cuda') for _ in range(T)]
st = torch.cuda.current_stream()
for host in (False, True, False, True):
    s.recycle_set(None)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record(st)
    reps = rk.solve_sequence(s, (lambda t: Bh[t]) if host else (lambda t: B[t]), T, 'hybrid', n_sw=3, host=host, x_out=Xh if host else X)
    e1.record(st); torch.cuda.synchronize(); wall = time.perf_counter() - t0
    sec = [r['seconds'] * 1e3 for r in reps]
    print('host' if host else 'dev ', 'events %.1f ms/sys' % (e0.elapsed_time(e1) / T), 'wall %.1f' % (wall * 1e3 / T),
          'rep.seconds mean %.2f' % np.mean(sec), 'rgcrot %.1f rbicg %.1f' % (np.mean(sec[:3]), np.mean(sec[3:])), flush=True)
