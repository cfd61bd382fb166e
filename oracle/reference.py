"""The unmodified reference ``phaseswe`` as a CPU checker and CPU baseline.

TEST INFRASTRUCTURE ONLY (same rule as ``pswe_oracle``): imported by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs, never by
the product package.

``oracle/build_ref.sh`` installs the reference with pip into ``oracle/_ref``
(git-ignored, travels to the GPU box); in this container the tree under
``/root/reference/pkg/src`` is used as a fallback.  ``load()`` returns the
``phaseswe`` module or None when neither exists.

``problem()`` turns one of our seeded cases into the reference's own objects
(``make_grid`` grid.py:81-107, ``PhysicsParams`` dynamics.py:34-63, ``State``
dynamics.py:72-118, ``kernel_weights`` averaging.py:80-106), so that the
reference's public ``averaged_tendency`` (averaging.py:116-156),
``step_averaged_ssprk3`` (integrator.py:83-103) and ``run``
(integrator.py:145-183) are called exactly as a user of the reference calls
them.
"""

from __future__ import annotations

import pathlib
import sys

HERE = pathlib.Path(__file__).resolve().parent
_CANDIDATES = (HERE / "_ref", pathlib.Path("/root/reference/pkg/src"))
_mod = None


def load():
    """The reference package, or None if it is not available on this machine."""
    global _mod
    if _mod is not None:
        return _mod
    for p in _CANDIDATES:
        if (p / "phaseswe" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import phaseswe
            _mod = phaseswe
            return _mod
    return None


def where() -> str | None:
    m = load()
    return None if m is None else str(pathlib.Path(m.__file__).resolve().parent)


class Problem:
    """A case restated in the reference's own types."""

    def __init__(self, ref, case):
        from phaseswe import averaging, dynamics, grid, propagator
        g = case.grid
        self.ref = ref
        self.grid = grid.make_grid(g.nx, g.ny, g.Lx, g.Ly)
        p = case.params
        self.params = dynamics.PhysicsParams(f=p.f, g=p.g, H=p.H, b=p.b)
        st = case.state
        self.state = dynamics.State(grid=self.grid, u=st.u, v=st.v, eta=st.eta, t=st.t)
        self.quadrature = averaging.kernel_weights(case.T_half, case.M)
        self.spec = propagator.PropagatorSpec.exact()
        self.case = case

    def sub_quadrature(self, m: int):
        """The 2m+1 central nodes of the case's quadrature with their weights
        renormalised to sum to 1 (a valid reference Quadrature): a bounded
        sample with the per-node work of the full evaluation."""
        import numpy as np
        from phaseswe import averaging
        q = self.quadrature
        M = q.M
        m = max(0, min(m, M - 1 if M > 0 else 0))
        s = np.array(q.s[M - m:M + m + 1])
        w = np.array(q.w[M - m:M + m + 1])
        w = w / float(w.sum())
        w = w / float(w.sum())
        w = 0.5 * (w + w[::-1])  # exactly symmetric after the rescale
        w = w / float(w.sum())
        return averaging.Quadrature(T=float(s[-1]) if m else 0.0, M=m, s=s, w=w)


def problem(case):
    ref = load()
    return None if ref is None else Problem(ref, case)
