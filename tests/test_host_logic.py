"""Host-side sequence controller (api.solve_sequence) on CPU, against a
recording stand-in for the librk solver: the pipelined host path stages
b_{t+1} before solving t, alternates the two staging slots, uploads a new
A epoch's bands before the solve that needs them, re-solves a switch-back
from the same slot, and synchronises the downloads once at the end; the
method schedule equals the one-call path's and the hybrid rule of P:662-669
(reading R16).  No GPU and no librk compute calls."""
import pytest
import torch

from paper_1501_03358_b200.api import solve_sequence


class _Op:
    def __init__(self, log):
        self.log = log

    def update_bands(self, bands):
        self.log.append(("bands", bands))


class _RecSolver:
    """Records the calls solve_sequence makes; solves 'fail' on demand."""

    def __init__(self, fail=()):
        self.log = []
        self.op = _Op(self.log)
        self.method = None
        self.fail = set(fail)
        self.staged = {}
        self.t = 0

    def _rep(self, converged):
        return {"krylov_matvecs": 10, "operator_applications": 1, "seconds": 0.0,
                "outcome": "CONVERGED" if converged else "MAX_MATVECS"}

    def set_method(self, m):
        self.method = m
        self.log.append(("method", m))

    def stage_rhs(self, slot, b):
        self.staged[slot] = int(b[0])
        self.log.append(("stage", slot, int(b[0])))

    def solve_staged(self, slot, x, tol=0.0):
        t = self.staged[slot]
        self.log.append(("solve", slot, t, self.method))
        x[0] = t
        ok = not (self.method == "rbicgstab" and t in self.fail)
        return x, self._rep(ok)

    def host_sync(self):
        self.log.append(("sync",))

    def solve_host(self, b, x, tol=0.0, x0_zero=False):
        t = int(b[0])
        self.log.append(("solve_host", t, self.method))
        x[0] = t
        ok = not (self.method == "rbicgstab" and t in self.fail)
        return x, self._rep(ok)


def _run(solver, n, pipeline, **kw):
    xs = [torch.zeros(4, dtype=torch.float64) for _ in range(n)]
    rhs = lambda t: torch.full((4,), float(t), dtype=torch.float64)
    reps = solve_sequence(solver, rhs, n, "hybrid", n_sw=2, epoch_of=lambda t: t // 3,
                          bands_for_epoch=lambda e: f"A{e}", host=True, x_out=xs,
                          pipeline=pipeline, **kw)
    return reps, xs


@pytest.mark.parametrize("kw", [{}, {"switchback": True}, {"refresh_on_epoch": True}])
def test_pipelined_controller_order(kw):
    n = 7
    s = _RecSolver(fail={4})
    reps, xs = _run(s, n, True, **kw)
    log = s.log
    # every x holds its own system's result
    assert [int(x[0]) for x in xs] == list(range(n))
    # staging: b_0 into slot 0 first, then b_{t+1} into slot (t+1) % 2 before solve t
    stages = [e for e in log if e[0] == "stage"]
    assert stages == [("stage", t % 2, t) for t in range(n)]
    for t in range(n):
        i_solve = next(i for i, e in enumerate(log) if e[0] == "solve" and e[2] == t)
        i_stage = log.index(("stage", t % 2, t))
        assert i_stage < i_solve
        if t + 1 < n:
            assert log.index(("stage", (t + 1) % 2, t + 1)) < i_solve
        # the slot a solve reads holds its own right-hand side
        assert log[i_solve][1] == t % 2
    # a new epoch's bands are uploaded before the first solve of that epoch
    for e in (1, 2):
        i_b = log.index(("bands", f"A{e}"))
        i_s = next(i for i, x in enumerate(log) if x[0] == "solve" and x[2] == 3 * e)
        assert i_b < i_s
    # one sync, at the end
    assert [e for e in log if e[0] == "sync"] == [("sync",)] and log[-1] == ("sync",)
    # switch-back re-solves system 4 by rGCROT from the same slot
    if kw.get("switchback"):
        assert reps[4]["tag"] == "rbicgstab+rgcrot"
        solves4 = [e for e in log if e[0] == "solve" and e[2] == 4]
        assert solves4 == [("solve", 0, 4, "rbicgstab"), ("solve", 0, 4, "rgcrot")]


@pytest.mark.parametrize("kw", [{}, {"switchback": True}, {"refresh_on_epoch": True},
                                {"refresh_every": 2}])
def test_pipelined_and_one_call_paths_agree(kw):
    """Same method schedule, tags and counts through both host paths."""
    a, xa = _run(_RecSolver(fail={4}), 8, True, **kw)
    b, xb = _run(_RecSolver(fail={4}), 8, False, **kw)
    assert [r["tag"] for r in a] == [r["tag"] for r in b]
    assert [r["krylov_matvecs"] for r in a] == [r["krylov_matvecs"] for r in b]
    assert all(torch.equal(x, y) for x, y in zip(xa, xb))
    # the hybrid rule: rGCROT for t < n_sw, then rBiCGStab (plus the policies)
    tags = [r["tag"] for r in a]
    assert tags[:2] == ["rgcrot", "rgcrot"]
    if not kw:
        assert tags[2:] == ["rbicgstab"] * 6
    if kw.get("refresh_on_epoch"):
        assert tags[3] == "rgcrot" and tags[6] == "rgcrot"
