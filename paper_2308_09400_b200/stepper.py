"""Projected-Newton time stepper with every per-iteration stage on the GPU.

Mirror of the reference's ``SolverConfig`` / ``StepStats`` / ``SimState`` / ``newton_step`` /
``advance_time_step`` (``/root/reference/pkg/src/tetipc/solver.py:32-235, :316-422``): the same
names, arguments, stopping rules and ``info`` / ``StepStats`` fields.  The state (x, v) and every
intermediate (contact table, blocks, matrix, gradient, direction) stay in HBM; per Newton iteration the
host sees a few scalars (contact counts, PCG result, CCD bound, one energy per line-search candidate).

``scene`` is duck-typed on the reference ``Scene`` (mesh.py:76-141): ``positions``,
``rest_positions``, ``masses``, ``fixed``, ``tets``, ``surf_tris``, ``surf_edges``, ``surf_verts``,
``gravity``, ``bbox_diagonal`` and, when ``materials`` is per body, ``bodies[i].tets``.
Only the GIPC mode is provided: the reference-IPC mode (finite-difference blocks + eigendecomposition)
is the baseline the paper replaces and is not on this path.
"""

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib, contacts, device, elasticity, friction, stencils
from .barrier import BarrierParams, c_params
from .solver import NewtonSystem

MODE_GIPC = "gipc"
MODE_REFERENCE = "reference-ipc"


@dataclass
class SolverConfig:
    """solver.py:32-51, field for field."""

    dt: float
    barrier: BarrierParams
    eps_d: float = 1e-2
    pcg_rel_tol: float = 1e-4
    pcg_max_iters: int = 2000
    newton_max_iters: int = 100
    friction_mu: float = 0.0
    friction_eps_v: float = 1e-3
    mode: str = MODE_GIPC
    accd_slack: float = 0.9
    line_search_floor: float = 1e-12
    mollify: bool = True
    # not in the reference: which preconditioner drives pcg_solve.  "block_jacobi" is the reference's
    # (solver.py:265-276); "mas" is the paper's alternative, domains re-ordered once per time
    # step.  Both stop on the reference's block-Jacobi-norm rule.  "auto" is the paper's "trial both and keep the
    # more efficient one": block-Jacobi until a solve of the current time step needs more than `auto_switch_iters`
    # iterations (MAS costs ~0.5 ms of setup and ~1.4 x per iteration, and takes ~3.3 x fewer iterations on
    # contact-dominated systems), MAS for the rest of that step.
    preconditioner: str = "block_jacobi"
    mas_levels: int = 1
    auto_switch_iters: int = 80

    def __post_init__(self):
        if self.dt <= 0.0 or self.eps_d <= 0.0 or self.pcg_rel_tol <= 0.0:
            raise ValueError("dt and tolerances must be positive")
        if self.mode not in (MODE_GIPC, MODE_REFERENCE):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.mode == MODE_REFERENCE:
            raise NotImplementedError("the reference-IPC baseline mode is not part of the GPU path")
        if self.preconditioner not in ("block_jacobi", "mas", "auto"):
            raise ValueError(f"unknown preconditioner {self.preconditioner!r}")


@dataclass
class StepStats:
    """solver.py:54-64."""

    step: int
    newton_iters: int
    pcg_iters: int
    min_distance: float
    energy: float
    alpha_min: float
    wall_ms: float
    converged: bool
    warning: str = ""


def _dev(a):
    """Device fp64 tensor of a host array; a device tensor passes through as the same object."""
    return device.to_device(a, np.float64)


def _tet_materials(scene, materials, nt):
    """Per-tet Lame parameters: per-body materials like solver.py:83-97, or one material / a
    (mu, lam) pair of arrays for scenes without a ``bodies`` list."""
    mu, lam = np.zeros(nt), np.zeros(nt)
    if hasattr(materials, "lame_mu"):
        mu[:], lam[:] = materials.lame_mu, materials.lame_lambda
    elif (isinstance(materials, (list, tuple)) and hasattr(scene, "bodies") and len(materials) == len(scene.bodies)
          and all(m is None or hasattr(m, "lame_mu") for m in materials)):   # not a (mu, lam) pair of arrays
        cursor = 0
        for i, body in enumerate(scene.bodies):
            k = int(np.asarray(body.tets).reshape(-1, 4).shape[0])
            if k == 0:
                continue
            if materials[i] is None:
                raise ValueError(f"body {i} has tets but no material")
            mu[cursor:cursor + k] = materials[i].lame_mu
            lam[cursor:cursor + k] = materials[i].lame_lambda
            cursor += k
    elif isinstance(materials, (list, tuple)) and len(materials) == 2 and not hasattr(materials[0], "lame_mu"):
        mu[:] = np.asarray(materials[0], dtype=np.float64)
        lam[:] = np.asarray(materials[1], dtype=np.float64)
    else:
        raise ValueError("materials: one per body, a single ElasticMaterial, or (mu, lam) per tet")
    return mu, lam


class SimState:
    """Device-resident simulation state (solver.py:67-235).  ``x`` and ``v`` are (N,3) device tensors;
    ``positions()`` / ``velocities()`` give host copies."""

    def __init__(self, scene, config, materials=None):
        t = device.torch()
        self.scene = scene
        self.config = config
        self.x = device.to_device(np.array(scene.positions, dtype=np.float64))
        self.v = t.zeros_like(self.x)
        self.n = int(self.x.shape[0])
        masses = np.asarray(scene.masses, dtype=np.float64)
        fixed = np.asarray(scene.fixed, dtype=bool)
        if np.any(masses[~fixed] <= 0.0):
            raise ValueError("free vertices need positive mass")
        self.masses, self.fixed = masses.copy(), fixed.copy()
        self.l = float(scene.bbox_diagonal)
        self.step_index = 0
        self.stats = []
        self._fixed_dev = device.to_device(fixed.astype(np.uint8)).bool()
        self._free_mass = device.to_device(np.where(fixed, 0.0, masses))[:, None]
        self._gravity = device.to_device(np.asarray(scene.gravity, dtype=np.float64).reshape(1, 3))
        self._rest = device.to_device(np.asarray(scene.rest_positions, dtype=np.float64))

        tets = np.asarray(scene.tets).reshape(-1, 4)
        self.tet_mesh = None
        if tets.shape[0]:
            mu, lam = _tet_materials(scene, materials, tets.shape[0])
            self.tet_mesh = elasticity.TetMesh(scene.rest_positions, tets, mu, lam)

        surf_verts = getattr(scene, "surf_verts", None)
        self.broad = contacts.BroadPhase(surf_verts, scene.surf_tris, scene.surf_edges, config.barrier.d_hat,
                                         np.asarray(scene.positions, dtype=np.float64))
        self.system = NewtonSystem(masses, fixed)
        self.friction_state = None
        self._last_detect = None
        self._mas_ordered = False
        self._auto_mas = False
        if config.friction_mu > 0.0:
            self._refresh_friction(self.x)

    def close(self):
        self.broad.close()
        self.system.close()

    def positions(self):
        return device.to_host(self.x)

    def velocities(self):
        return device.to_host(self.v)

    # -- contact set (solver.py:112-116) ----------------------------------------------------
    def detect(self, x, candidates=None):
        """``DeviceStencilTable`` of every stencil closer than d_hat, in the reference's list order.

        The reference detects at the accepted line-search candidate and again, on the same positions, at
        the top of the next Newton iteration and at the end of the step (solver.py:324, :343, :400); the
        last result is kept and returned when the very same, unmodified tensor comes back.  ``candidates``:
        (vt, ee) known to contain every pair within d_hat at ``x`` (the swept join of the step this ``x``
        lies on): the broad phase is skipped, the list is the same (any superset of candidates gives it)."""
        last = self._last_detect
        if last is not None and last[0] is x and last[1] == x._version:
            return last[2]
        promote = self.config.mollify and self.config.mode == MODE_GIPC
        vt, ee = candidates if candidates is not None else self.broad.query(x)
        table, extra = contacts.narrow_phase_device(x, self._rest, vt, ee, self.config.barrier.d_hat,
                                                    promote_parallel=promote, want_origin=False)
        table.kind_dev = extra.kind
        self._last_detect = (x, x._version, table)
        return table

    # -- energies (solver.py:118-175) --------------------------------------------------------
    def _inertia_target(self, x0):
        cfg = self.config
        x0 = _dev(x0)
        x_tilde = x0 + cfg.dt * _dev(self.v) + cfg.dt ** 2 * self._gravity
        x_tilde[self._fixed_dev] = x0[self._fixed_dev]
        return x_tilde

    def _barrier_energy(self, x, table):
        return stencils.barrier_energy(table, x, self.config.barrier) if table.n else 0.0

    def _friction_energy(self, x, x_start):
        if self.friction_state is None or self.friction_state.n == 0:
            return 0.0
        return friction.evaluate(self.friction_state, x, x_start, want_grad=False, want_hess=False).total_energy()

    def _elastic_energy(self, x):
        if self.tet_mesh is None:
            return 0.0
        energy, _ = self.tet_mesh.evaluate(x, want_grad=False, want_hess=False)
        return float(energy.sum().item())

    def evaluate_energy(self, x, x_tilde, x_start, stencils=None, candidates=None):
        """Incremental potential at x; detects contacts unless a table is given (``candidates``: see ``detect``)."""
        x, x_tilde, x_start = _dev(x), _dev(x_tilde), _dev(x_start)
        table = self.detect(x, candidates) if stencils is None else stencils
        dx = x - x_tilde
        inertia = 0.5 * float((self._free_mass * dx * dx).sum().item())
        dt2 = self.config.dt ** 2
        return inertia + dt2 * (self._elastic_energy(x) + self._barrier_energy(x, table)
                                + self._friction_energy(x, x_start))

    # -- gradient and PSD blocks (solver.py:177-235) -----------------------------------------
    def assemble_local_quadratics(self, x, x_start, table):
        """dt^2-scaled families in the reference's block order: elastic, barrier, friction.
        Returns a list of ``stencils.Family`` (device tensors), at most seven."""
        dt = self.config.dt
        fams = []
        if self.tet_mesh is not None:
            fams.append(self.tet_mesh.evaluate(x, dt=dt, want_energy=False)[1])
        if table.n:
            batch = stencils.evaluate(table, x, self.config.barrier, dt=dt, want_energy=False)
            batch.raise_on_penetration()   # _barrier_block -> build_diagonal_jacobian raises on d2 <= 0 (gap.py:61)
            fams += [batch.families[s] for s in sorted(batch.families)]
        if self.friction_state is not None and self.friction_state.n:
            fb = friction.evaluate(self.friction_state, x, x_start, want_energy=False)
            fams += [fb.families[s] for s in sorted(fb.families)]
        return fams

    def gradient(self, x, x_tilde, fams):
        return self.system.gradient(x, x_tilde, [f.grad for f in fams])

    def _refresh_friction(self, x, table=None):
        if table is None:
            table = self.detect(x)
        cfg = self.config
        self.friction_state = friction.update_state(table, x, cfg.friction_mu, cfg.friction_eps_v, cfg.dt,
                                                    params=cfg.barrier)

    def min_distance(self, x, table):
        """sqrt(min d2) over a contact table (advance_time_step's end-of-step report); NaN when empty."""
        if table.n == 0:
            return float("nan")
        d2 = device.empty((table.n,))
        prm = c_params(self.config.barrier)
        null = C.c_void_p()
        _lib.check(_lib.lib().b200ipc_diagonal_jacobian(
            prm, self.n, device.ptr(x), table.n, device.ptr(table.kind_dev), device.ptr(table.verts),
            device.ptr(table.sub), device.ptr(d2), null, null, null, null, null, null, null, null, null,
            device.stream()), "diagonal_jacobian")
        return float(np.sqrt(d2.min().item()))


def _search_direction(state, x, x_tilde, x_start, table):
    """Newton direction at x on the device: blocks -> BSR matrix -> gradient -> block-Jacobi PCG, fixed rows
    zeroed (solver.py:325-334).  Returns (direction (N,3) tensor, PCG iterations, PCG converged)."""
    cfg = state.config
    only_barrier = state.tet_mesh is None and not (state.friction_state is not None and state.friction_state.n)
    if only_barrier and table.n and state.system.factors_fit({s: table.family_count(s) for s in (2, 3, 4)}):
        # barrier blocks are rank one: assemble straight from the factors z, the dense blocks are never written
        # (bitwise the same matrix, b200ipc_assemble_numeric_factors)
        batch = stencils.evaluate(table, x, cfg.barrier, dt=cfg.dt, want_energy=False, want_hess=False, want_factors=True)
        batch.raise_on_penetration()
        fams = [batch.families[s] for s in sorted(batch.families)]
        state.system.set_pattern([(f.s, f.vids) for f in fams])
        state.system.assemble_from_factors([f.fac for f in fams])
    else:
        fams = state.assemble_local_quadratics(x, x_start, table)
        state.system.set_pattern([(f.s, f.vids) for f in fams])
        state.system.assemble([f.hess for f in fams])
    rhs = -state.gradient(x, x_tilde, fams)
    prec = cfg.preconditioner
    if prec == "auto":
        prec = "mas" if state._auto_mas else "block_jacobi"
    if prec == "mas" and not state._mas_ordered:
        state.system.mas_order(x)          # once per time step: positions move by a fraction of d_hat per iteration
        state._mas_ordered = True
    flat, iters, ok, _, _ = state.system.pcg(rhs, cfg.pcg_rel_tol, cfg.pcg_max_iters,
                                             preconditioner=prec, mas_levels=cfg.mas_levels)
    if cfg.preconditioner == "auto" and prec == "block_jacobi" and iters > cfg.auto_switch_iters:
        state._auto_mas = True
    direction = flat.view(-1, 3)
    direction[state._fixed_dev] = 0.0
    return direction, iters, ok


def _backtrack(state, x, direction, alpha, x_tilde, x_start, energy_prev, candidates=None):
    """Halve alpha from the CCD bound until the incremental potential does not rise, contacts re-detected
    at every candidate (solver.py:342-351).  Returns (x_new, energy_new, alpha) or None on collapse.
    ``candidates``: the swept join of the step (every trial x + alpha d, alpha <= 1, lies inside it)."""
    floor = state.config.line_search_floor
    while alpha >= floor:
        trial = x + alpha * direction
        energy = state.evaluate_energy(trial, x_tilde, x_start, candidates=candidates if alpha <= 1.0 else None)
        if energy <= energy_prev:
            return trial, energy, alpha
        alpha *= 0.5
    return None


def newton_step(state, x, x_tilde, x_start, energy_prev):
    """One projected-Newton iteration with CCD-bounded backtracking (solver.py:316-362).

    Returns (x_new, energy_new, info) with the reference's ``info`` keys; a collapsed line search returns
    the input iterate with ``accepted`` False and ``alpha`` 0.
    """
    x, x_tilde, x_start = _dev(x), _dev(x_tilde), _dev(x_start)
    table = state.detect(x)
    direction, pcg_iters, pcg_ok = _search_direction(state, x, x_tilde, x_start, table)
    # ONE swept join per Newton iteration: boxes over x and x + d grown by 0.51 d_hat contain every pair that is
    # within d_hat anywhere on the step, so the list serves (a) the CCD filter, after the reference's own
    # swept-box test at 1e-3 d_hat has cut it down to sweep_candidates' exact set (proximity.py:388-421), and
    # (b) the contact detection of every line-search candidate, which then skips its broad phase.  Same bound,
    # same contact lists; one grid join instead of two.
    d_hat = state.config.barrier.d_hat
    swept = state.broad.sweep(x, direction, margin=0.51 * d_hat)
    bound = contacts.ccd_filter_superset_device(swept[0], swept[1], x, direction, 1e-3 * d_hat,
                                                slack=state.config.accd_slack)
    found = _backtrack(state, x, direction, min(1.0, bound), x_tilde, x_start, energy_prev, candidates=swept)
    info = {"pcg_iters": pcg_iters, "pcg_converged": pcg_ok, "alpha": 0.0, "accepted": found is not None,
            "d_inf": float(direction.abs().max().item()) if direction.numel() else 0.0, "n_contacts": table.n}
    if found is None:
        return x, energy_prev, info
    info["alpha"] = found[2]
    return found[0], found[1], info


def advance_time_step(state):
    """One time step: Newton iterations until |d|_inf / (l dt) <= eps_d, at least one, at most
    ``newton_max_iters`` ("newton-cap"); a collapsed line search ends the step ("line-search-collapse").
    Then velocities, the end-of-step contact set, the friction refresh and the ``StepStats`` record
    (solver.py:365-422)."""
    cfg = state.config
    clock = time.perf_counter()
    state.x, state.v = _dev(state.x), _dev(state.v)      # host arrays assigned by the caller are welcome
    x_start = state.x        # iterates are never modified in place: no copies, and detect's cache applies
    state._mas_ordered = False   # MAS domains follow the positions at the start of the step
    state._auto_mas = False      # "auto" starts every step with the reference's preconditioner
    x_tilde = state._inertia_target(x_start)
    x, energy = x_start, state.evaluate_energy(x_start, x_tilde, x_start)

    tally = {"newton": 0, "pcg": 0, "alpha_min": 1.0}
    outcome = "newton-cap"
    for _ in range(cfg.newton_max_iters):
        x, energy, info = newton_step(state, x, x_tilde, x_start, energy)
        tally["newton"] += 1
        tally["pcg"] += info["pcg_iters"]
        if not info["accepted"]:
            outcome = "line-search-collapse"
            break
        tally["alpha_min"] = min(tally["alpha_min"], info["alpha"])
        if info["d_inf"] / (state.l * cfg.dt) <= cfg.eps_d:     # the reference's expression, rounding included
            outcome = ""
            break

    velocity = (x - x_start) / cfg.dt
    velocity[state._fixed_dev] = 0.0
    state.x, state.v = x, velocity
    state.step_index += 1

    closing = state.detect(x)
    if cfg.friction_mu > 0.0:
        state._refresh_friction(x, closing)

    stats = StepStats(step=state.step_index, newton_iters=tally["newton"], pcg_iters=tally["pcg"],
                      min_distance=state.min_distance(x, closing), energy=energy, alpha_min=tally["alpha_min"],
                      wall_ms=(time.perf_counter() - clock) * 1e3, converged=outcome == "", warning=outcome)
    state.stats.append(stats)
    return stats
