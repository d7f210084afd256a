"""BASELINE.json configs as concrete workloads (operator + RHS recipe +
solver parameters).  Parameter readings:

* Jacobi(5+1) preconditioner everywhere, omega_l = 0.8, omega_g = 1.0 (D9, D10)
* k_t = max(k - 10, ceil(k/2)) (D12; "k-10")
* p1 (inner vectors selected per cycle) = 1 for channel-shaped c1/c2/c4,
  2 for porous-shaped c3/c5 (D13)
* tol = 1e-8 on ||b - A x|| / ||b|| (D4), max 2000 Krylov matvecs (D19)
* hybrid switch after n_sw = 3 rGCROT systems (BASELINE configs[2]/[4])
"""
import math
from dataclasses import dataclass, field, replace

from .stencils import channel19, convection_diffusion_c1, porous7


@dataclass(frozen=True)
class SolverParams:
    method: str = "rgcrot"       # rgcrot | gmres | bicgstab | rbicgstab | hybrid
    m: int = 20
    k_max: int = 10
    k_t: int = 5
    p1: int = 1
    n_sw: int = 3
    tol: float = 1e-8
    max_mv: int = 2000
    trunc: str = "T1"
    ortho: str = "cgs2"          # oracle: cgs2 (D8, block CGS applied twice) | mgs (Alg. 3 literal)
    sweeps: int = 5
    omega_l: float = 0.8
    omega_g: float = 1.0
    divergence: float = 1e4
    zblocks: int = 1             # block-Jacobi z-blocks of the local sweeps (1 = global, R17)
    precond: str = "jacobi"      # jacobi | ssor (multicolour, R18) | none
    omega_s: float = 1.0         # SSOR relaxation (SPEC S:106 default)


def k_trunc(k):
    return max(k - 10, int(math.ceil(k / 2)))


@dataclass
class Workload:
    name: str
    make_problem: object = field(repr=False)
    params: SolverParams
    n_systems: int
    epoch_every: int = 0          # 0: A constant; else epoch = t // epoch_every
    description: str = ""

    def problem(self):
        return self.make_problem()

    def epoch(self, t):
        return t // self.epoch_every if self.epoch_every else 0


def _rg(m, k, p1):
    return SolverParams(method="rgcrot", m=m, k_max=k, k_t=k_trunc(k), p1=p1)


def _hy(m, k, p1, n_sw=3):
    return SolverParams(method="hybrid", m=m, k_max=k, k_t=k_trunc(k), p1=p1, n_sw=n_sw)


WORKLOADS = {
    # BASELINE.json configs[0..4]
    "c1": Workload("c1", lambda: convection_diffusion_c1(16), _rg(20, 10, 1), 1,
                   description="16^3 7-pt convection-diffusion, rGCROT(20,10), 1 RHS"),
    "c2": Workload("c2", lambda: channel19(64), _rg(30, 20, 1), 10,
                   description="64^3 19-pt channel, rGCROT(30,20), 10 RHS, A constant"),
    "c3": Workload("c3", lambda: porous7(128, 6), _hy(10, 20, 2), 20,
                   description="128^3 7-pt porous, hybrid(3) rGCROT(10,20)->rBiCGStab, 20 RHS"),
    # c4 truncates by principal angles (T2, reading R13): "GCROT measures
    # angles between successive search spaces" -- measured on c4,
    # 448 vs 480 Krylov matvecs per system for T1 (profiles/r02_compare/)
    "c4": Workload("c4", lambda: channel19(256), replace(_rg(40, 30, 1), trunc="T2"), 50, epoch_every=10,
                   description="256^3 19-pt channel, rGCROT(40,30) T2, 50 RHS, A perturbed every 10"),
    "c4h": Workload("c4h", lambda: channel19(256), replace(_hy(40, 30, 1), trunc="T2"), 50, epoch_every=10,
                    description="256^3 19-pt channel, hybrid(3) comparison arm of c4"),
    "c5": Workload("c5", lambda: porous7(512, 12), _hy(10, 20, 2), 20,
                   description="512^3 7-pt porous r=12, hybrid(3), 20 RHS"),
    # shrunken analogues (oracle finishes in seconds; parity tests)
    "c1s": Workload("c1s", lambda: convection_diffusion_c1(8), _rg(10, 6, 1), 1),
    "c2s": Workload("c2s", lambda: channel19(16), _rg(12, 8, 1), 6),
    "c3s": Workload("c3s", lambda: porous7(24, 3), _hy(8, 8, 2), 8),
    # 32^3: the smallest porous grid the fused TMA chain tiles (nx % 32, ny % 16)
    "c3m": Workload("c3m", lambda: porous7(32, 3), _hy(8, 8, 2), 6),
    "c4s": Workload("c4s", lambda: channel19(16), _rg(12, 10, 1), 9, epoch_every=3),
    # 32^3 channel: the smallest 19-point grid the fused 19-point chain tiles
    # (nx % 32, ny % 8, nz >= 16); hybrid with A epochs (tests, smoke)
    "c2m": Workload("c2m", lambda: channel19(32), _hy(12, 8, 1, n_sw=2), 4, epoch_every=2),
    "c4hs": Workload("c4hs", lambda: channel19(16), _hy(12, 10, 1), 9, epoch_every=3),
    # 64^3 analogues of c4 with c4's solver parameters (the oracle runs whole
    # sequences in ~1 h; diagnosis of the c4 hybrid, profiles/r02_c4h_diag/)
    "c4m": Workload("c4m", lambda: channel19(64), _rg(40, 30, 1), 30, epoch_every=10,
                    description="64^3 19-pt channel, rGCROT(40,30), 30 RHS, A perturbed every 10"),
    "c4hm": Workload("c4hm", lambda: channel19(64), _hy(40, 30, 1), 30, epoch_every=10,
                     description="64^3 19-pt channel, hybrid(3) rGCROT(40,30)->rBiCGStab, 30 RHS"),
}


def get_workload(name, **overrides):
    w = WORKLOADS[name]
    if overrides:
        w = Workload(w.name, w.make_problem, replace(w.params, **overrides),
                     w.n_systems, w.epoch_every, w.description)
    return w


def slab_range(nz, rank, nranks):
    """z-slab decomposition: rank p owns planes [p*nz/P, (p+1)*nz/P)."""
    return (rank * nz) // nranks, ((rank + 1) * nz) // nranks
