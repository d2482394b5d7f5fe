"""The drop-in as code: the reference package ``tetipc`` running UNMODIFIED on this backend.

Two levels, both described in INTEGRATION.md:

1. ``kernel_backend(tetipc)`` -- the reference's own plugin seam
   (``/root/reference/pkg/src/tetipc/kernels/__init__.py:13-32``): the five module-level functions
   ``pt_classify_batch, ee_classify_batch, cross_sq_batch, matvec_blocks, accd_max_step`` and ``BACKEND`` are
   pointed at ``paper_2308_09400_b200.kernels`` (ctypes over libb200ipc.so).  Everything above the seam --
   ``proximity.py``, ``gap.py``, ``solver.py`` -- is the reference's code, untouched.
2. ``b200_sim_state(tetipc)`` -- a subclass of the reference's ``SimState`` (``solver.py:67-235``) whose
   per-stencil Python loops (``detect``, ``_barrier_energy``, ``barrier_gradient_blocks``, the barrier loop of
   ``assemble_local_quadratics``) are replaced by the batched device entry points, with the reference's
   signatures and return types; ``batched_solver(tetipc)`` additionally routes ``pcg_solve`` /
   ``sweep_candidates`` / ``global_ccd_filter`` (``solver.py:331-340``) to the device.  The reference's own
   ``newton_step`` / ``advance_time_step`` (``solver.py:318-422``) run unmodified on top.

``tetipc`` itself is never imported by the product path: callers pass the module in (tests find it under
``/root/reference/pkg/src`` or ``baseline/_ref``).  There is no CPU fallback here either: every replaced
function goes to the GPU or raises.
"""

import contextlib

import numpy as np

from . import contacts, kernels as b200_kernels, proximity as bprox, solver as bsolver, stencils
from .barrier import BarrierParams

_SEAM = ("pt_classify_batch", "ee_classify_batch", "cross_sq_batch", "matvec_blocks", "accd_max_step")


@contextlib.contextmanager
def kernel_backend(tetipc):
    """Within the block ``tetipc.kernels`` dispatches to the B200 backend (``BACKEND == "b200"``)."""
    seam = tetipc.kernels
    saved = {name: getattr(seam, name) for name in _SEAM + ("BACKEND",)}
    try:
        for name in _SEAM:
            setattr(seam, name, getattr(b200_kernels, name))
        seam.BACKEND = b200_kernels.BACKEND
        yield seam
    finally:
        for name, fn in saved.items():
            setattr(seam, name, fn)


def barrier_params(ref_params):
    """The reference's ``BarrierParams`` (barrier.py:24-53) as this package's, field for field."""
    if isinstance(ref_params, BarrierParams):
        return ref_params
    return BarrierParams(d_hat=ref_params.d_hat, kappa=ref_params.kappa, d_thr_ratio=ref_params.d_thr_ratio,
                         use_filter=ref_params.use_filter, form=ref_params.form)


def to_reference_stencils(tetipc, table):
    """Host ``StencilTable`` -> the reference's own ``ContactStencil`` objects, in list order."""
    rp = tetipc.proximity
    out = []
    for st in table.to_stencils():
        out.append(rp.ContactStencil(kind=rp.StencilKind(st.kind.value), verts=st.verts, eps_x=st.eps_x,
                                     edge_pair=st.edge_pair, sub=st.sub, origin=st.origin))
    return out


def b200_sim_state(tetipc):
    """``class B200SimState(tetipc.solver.SimState)``: same constructor, same method signatures and return
    types; contact detection and every per-stencil barrier loop batched on the GPU."""
    ref = tetipc.solver

    class B200SimState(ref.SimState):
        def _table(self, stencils_):
            return bprox.StencilTable.from_stencils(stencils_)

        def detect(self, x):                                             # solver.py:116-118
            promote = self.config.mollify and self.config.mode == ref.MODE_GIPC
            if self.config.mode != ref.MODE_GIPC:
                return super().detect(x)
            x = np.asarray(x, dtype=np.float64)
            d_hat = self.config.barrier.d_hat
            bp = contacts.BroadPhase(getattr(self.scene, "surf_verts", None), self.scene.surf_tris,
                                     self.scene.surf_edges, d_hat, x)
            try:
                vt, ee = bp.query(x)
                table = contacts.narrow_phase(x, self.scene.rest_positions, vt, ee, d_hat, promote)
            finally:
                bp.close()
            return to_reference_stencils(tetipc, table)

        def _barrier_energy(self, x, stencils_):                         # solver.py:127-146
            if self.config.mode != ref.MODE_GIPC or not stencils_:
                return super()._barrier_energy(x, stencils_)
            try:
                return stencils.barrier_energy(self._table(stencils_), x, barrier_params(self.config.barrier))
            except Exception as exc:                                     # same class the reference raises
                if type(exc).__name__ == "InterpenetrationError":
                    raise tetipc.gap.InterpenetrationError(str(exc)) from exc
                raise

        def barrier_gradient_blocks(self, x, stencils_):                 # solver.py:186-188 (raw gradients)
            if self.config.mode != ref.MODE_GIPC or not stencils_:
                return super().barrier_gradient_blocks(x, stencils_)
            batch = stencils.evaluate(self._table(stencils_), x, barrier_params(self.config.barrier), dt=1.0,
                                      want_hess=False)
            batch.raise_on_penetration()
            blocks = batch.to_local_quadratics(keep_inactive=True)
            return [blk.grad for blk in blocks]

        def assemble_local_quadratics(self, x, x_start, stencils_):      # solver.py:190-216
            if self.config.mode != ref.MODE_GIPC:
                return super().assemble_local_quadratics(x, x_start, stencils_)
            rest = super().assemble_local_quadratics(x, x_start, [])     # elastic and friction loops, unchanged
            n_el = self.scene.tets.shape[0]
            if not stencils_:
                return rest
            batch = stencils.evaluate(self._table(stencils_), x, barrier_params(self.config.barrier),
                                      dt=self.config.dt)
            batch.raise_on_penetration()
            LQ = tetipc.barrier.LocalQuadratic
            mine = [LQ(vert_ids=b.vert_ids, grad=b.grad, hess=b.hess) for b in batch.to_local_quadratics()]
            # reference order: elastic, barrier (list order, inactive rows dropped), friction
            return rest[:n_el] + mine + rest[n_el:]

    return B200SimState


@contextlib.contextmanager
def batched_solver(tetipc):
    """Within the block the reference's ``newton_step`` solves and filters on the device:
    ``solver.pcg_solve`` -> assembled BSR + persistent PCG kernel (same arguments and return tuple),
    ``proximity.sweep_candidates`` / ``global_ccd_filter`` -> grid join + ACCD kernel."""
    ref, rp = tetipc.solver, tetipc.proximity
    saved = (ref.pcg_solve, rp.sweep_candidates, rp.global_ccd_filter)
    try:
        ref.pcg_solve = bsolver.pcg_solve
        rp.sweep_candidates = contacts.sweep_candidates
        rp.global_ccd_filter = contacts.global_ccd_filter
        yield
    finally:
        ref.pcg_solve, rp.sweep_candidates, rp.global_ccd_filter = saved
