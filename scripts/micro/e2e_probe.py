import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1501_03358_b200 as rk
from problems import get_workload
w = get_workload('c3'); prm = w.params; prob = w.problem()
ctx = rk.Context(0)
op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets, torch.from_numpy(prob.bands()).cuda(), prob.periodic)
s = rk.Solver(op, rk.config_from_params(prm))
T = 6
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
    print('host' if host else 'dev ', 'events %.1f ms' % e0.elapsed_time(e1), 'wall %.1f ms' % (wall*1e3), [r['krylov_matvecs'] for r in reps], 'rep.seconds sum %.1f ms' % (1e3*sum(r['seconds'] for r in reps)))
# raw copy speed
a = torch.empty(prob.N, dtype=torch.float64, device='cuda')
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(10): a.copy_(Bh[0], non_blocking=True)
e1.record(st); torch.cuda.synchronize(); print('H2D 16 MiB pinned: %.3f ms' % (e0.elapsed_time(e1)/10))
