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


# ---------------------------------------------------------------------------------------------------------------
# 3. function overlay: every function of the reference's modules that this package mirrors, swapped in place
# ---------------------------------------------------------------------------------------------------------------
# (reference module, name) -> the mirror.  Arguments are duck-typed on the reference's field names, so the
# reference's own objects (ContactStencil, BarrierParams, DiagonalJacobian, FrictionDatum, Scene ...) go straight in;
# results and exceptions are handed back as the REFERENCE's classes.

def _overlay_table():
    from . import barrier, elasticity, friction, gap, mollifier

    return {
        "barrier": {n: getattr(barrier, n) for n in ("barrier_value", "barrier_dg", "barrier_d2g", "lambda1", "lambda23",
                                                      "filtered_lambda1", "build_local_quadratic")},
        "gap": {n: getattr(gap, n) for n in ("build_diagonal_jacobian", "gap_function")},
        "proximity": {"stencil_distance": gap.stencil_distance, "parallel_measure": gap.parallel_measure,
                      "find_contact_pairs": contacts.find_contact_pairs, "accd_step_bound": contacts.accd_step_bound,
                      "sweep_candidates": contacts.sweep_candidates, "global_ccd_filter": contacts.global_ccd_filter},
        "mollifier": {n: getattr(mollifier, n) for n in ("mollified_eigensystem", "mollified_barrier_value",
                                                          "mollified_gradient", "build_mollified_local_quadratic")},
        "friction": {n: getattr(friction, n) for n in ("f0_f1", "potential", "friction_force", "friction_hessian_psd",
                                                        "tangential_displacement", "update_friction_state")},
        "elasticity": {n: getattr(elasticity, n) for n in ("rest_data", "batch_grad_hess", "tet_energy_grad_hess")},
        "solver": {n: getattr(bsolver, n) for n in ("group_blocks", "matvec_matrix_free", "block_jacobi_preconditioner",
                                                    "pcg_solve")},
        "kernels": {n: getattr(b200_kernels, n) for n in _SEAM},
    }


def _reference_classes(tetipc):
    """name -> class for every dataclass / enum / exception the reference's modules define."""
    import enum
    import importlib

    out = {}
    for mod in ("proximity", "gap", "barrier", "mollifier", "friction", "elasticity"):
        m = importlib.import_module(f"{tetipc.__name__}.{mod}")
        for name, val in vars(m).items():
            if isinstance(val, type) and val.__module__ == m.__name__ and (
                    hasattr(val, "__dataclass_fields__") or issubclass(val, (enum.Enum, Exception))):
                out[name] = val
    return out


def _as_reference(obj, classes):
    """This package's records / enums -> the reference's classes of the same name (recursively through lists,
    tuples and record fields); arrays and scalars pass through."""
    import dataclasses
    import enum

    if isinstance(obj, list):
        return [_as_reference(o, classes) for o in obj]
    if type(obj) is tuple:
        return tuple(_as_reference(o, classes) for o in obj)
    cls = classes.get(type(obj).__name__)
    if cls is None or isinstance(obj, cls) or not type(obj).__module__.startswith(__package__):
        return obj
    if isinstance(obj, enum.Enum):
        return cls(obj.value)
    if dataclasses.is_dataclass(obj):
        return cls(**{f.name: _as_reference(getattr(obj, f.name), classes) for f in dataclasses.fields(cls)
                      if hasattr(obj, f.name)})
    return obj


@contextlib.contextmanager
def function_overlay(tetipc, calls=None, batched=False):
    """Within the block every function of ``tetipc.{barrier, gap, proximity, mollifier, friction, elasticity,
    solver, kernels}`` that this package mirrors IS the mirror -- in the defining module and in every other
    ``tetipc`` module that imported it by name -- so the reference's own callers and its own test-suite
    (``tests/test_gpu_reference_suite.py``) exercise the B200 backend.  ``calls``: optional dict, filled with
    ``"module.function" -> number of calls``.  ``batched``: additionally ``tetipc.solver.SimState`` IS
    ``b200_sim_state(tetipc)`` (contact detection and the per-stencil barrier loops as single batched launches)."""
    import functools
    import importlib
    import sys

    classes = _reference_classes(tetipc)
    root = tetipc.__name__

    def wrap(key, fn):
        @functools.wraps(fn)
        def mirrored(*args, **kwargs):
            if calls is not None:
                calls[key] = calls.get(key, 0) + 1
            try:
                return _as_reference(fn(*args, **kwargs), classes)
            except Exception as exc:
                cls = classes.get(type(exc).__name__)
                if (cls is not None and not isinstance(exc, cls) and isinstance(cls, type)
                        and issubclass(cls, Exception) and type(exc).__module__.startswith(__package__)):
                    raise cls(*exc.args) from exc
                raise
        return mirrored

    saved = []
    try:
        for mod, table in _overlay_table().items():
            ref_mod = importlib.import_module(f"{root}.{mod}")
            for name, fn in table.items():
                orig = getattr(ref_mod, name)
                new = wrap(f"{mod}.{name}", fn)
                for mname, m in list(sys.modules.items()):
                    if m is None or not (mname == root or mname.startswith(root + ".")):
                        continue
                    for attr, val in list(vars(m).items()):
                        if val is orig:
                            saved.append((m, attr, orig))
                            setattr(m, attr, new)
        if batched:
            solver_mod = importlib.import_module(f"{root}.solver")
            orig_cls = solver_mod.SimState
            new_cls = b200_sim_state(tetipc)
            if calls is not None:
                for meth in ("detect", "_barrier_energy", "barrier_gradient_blocks", "assemble_local_quadratics"):
                    def counted(self, *a, _m=getattr(new_cls, meth), _k="SimState." + meth, **kw):
                        calls[_k] = calls.get(_k, 0) + 1
                        return _m(self, *a, **kw)
                    setattr(new_cls, meth, counted)
            for mname, m in list(sys.modules.items()):
                if m is not None and (mname == root or mname.startswith(root + ".")):
                    for attr, val in list(vars(m).items()):
                        if val is orig_cls:
                            saved.append((m, attr, orig_cls))
                            setattr(m, attr, new_cls)
        kernels_mod = importlib.import_module(f"{root}.kernels")
        saved.append((kernels_mod, "BACKEND", kernels_mod.BACKEND))
        kernels_mod.BACKEND = b200_kernels.BACKEND
        yield
    finally:
        for m, attr, orig in reversed(saved):
            setattr(m, attr, orig)
