#!/usr/bin/env python
"""Benchmark of the GIPC barrier hot path on B200 (contract: see DESIGN.md "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Headline (BASELINE.json metric, configs[1]): PSD barrier Hessian stencils/s, fp64, on the
nearly-parallel edge-edge stress set (1M EE queries -> mollified EEpar/PEpar/PPpar stencils plus
the plain rows the recipe mixes in).  One *step* = one evaluation of the whole kind-sorted stencil
table: energy + gradient + analytically PSD-projected Hessian block per stencil, written as the
dense 12x12 / 9x9 / 6x6 families the reference's ``group_blocks`` produces.  The second half of the
metric ("assembly+SpMV ms per Newton step") is measured on a teaser-style cloth stack (~1M
contacts) and reported under "newton".

Timing: W untimed warm-up steps, then K steps between CUDA events on the launching stream,
bracketed by barrier + synchronize; max over ranks.  Every step rewrites 1.27 GB of blocks, ten
times the 126 MB L2, so no flush is needed ("l2" in config).  N > 1 runs N independent replicas
(one scene per GPU, no data-path collective): weak scaling.  ``python bench.py --gpus N`` without a
rank environment re-executes itself under ``torch.distributed.run`` with N ranks
(``scene_batch.launch``); under torchrun it joins the ranks it is given.  ``--dry-run`` rehearses that
launch / aggregate path on CPUs with gloo (tests/test_multiproc.py).

``--impl reference`` times the CPU implementation of the same path on the SAME workload table (the same
1 M-row config-2 table, same config object) and prints the same ``newton`` keys, measured with the
reference's own compiled ``matvec_blocks`` (oracle/_ref) inside the reference's PCG recurrence.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PSD barrier Hessian stencils/s (fp64)"
UNIT = "stencils/s"
BYTES_PER_STENCIL = {4: 1272, 3: 740, 2: 352}  # verts + energy + grad + hess (parallel: +9)
KIND_SIZE = np.array([4, 4, 3, 4, 2, 4, 4])
KIND_PAR = np.array([0, 1, 0, 1, 0, 1, 0])


def algorithmic_bytes(kind_off, n_positions):
    """per stencil 4s (verts) [+9 parallel] + 8 (energy) + 24s (grad) + 72s^2 (hess),
    plus every referenced vertex position once (24 B each)."""
    counts = np.diff(np.asarray(kind_off))
    per = np.array([BYTES_PER_STENCIL[int(s)] for s in KIND_SIZE]) + 9 * KIND_PAR
    return int((counts * per).sum()) + 24 * int(n_positions)


def measured_peak():
    """HBM peak for the roofline: the driver-written MEASURED_PEAKS.json when present (key `hbm_gbs`;
    otherwise the sustained, then any, HBM GB/s figure it holds), else the recipe's fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        flat = {}

        def walk(prefix, node):
            if isinstance(node, dict):
                for k, v in node.items():
                    walk(f"{prefix}.{k}" if prefix else str(k), v)
            elif isinstance(node, (int, float)) and not isinstance(node, bool):
                flat[prefix.lower()] = float(node)

        walk("", data)
        if "hbm_gbs" in flat:
            return flat["hbm_gbs"], "measured (MEASURED_PEAKS.json hbm_gbs)"
        hbm = {k: v for k, v in flat.items() if "hbm" in k and v > 100.0}
        for want in ("sustain", ""):
            for k in sorted(hbm):
                if want in k:
                    return hbm[k], f"measured (MEASURED_PEAKS.json {k})"
    except (OSError, ValueError, TypeError):
        pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.rows, self.proc, self.index = [], None, index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            if len(r) < 7:
                continue
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for name, val in zip(names, r[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def time_steps(torch, fn, steps, warmup, dist=None):
    """The contract's timed region (scene_batch.timed_steps): ms for all ``steps`` on this rank."""
    from paper_2308_09400_b200 import scene_batch

    return scene_batch.timed_steps(fn, steps, warmup, dist, cuda=True)


def workload_config(n, kinds, world, alg_bytes):
    """The ``config`` object of BOTH arms (the driver compares them): BASELINE configs[1]."""
    return {"workload": "config2-parallel-ee: 1M nearly-parallel edge-edge queries (BASELINE configs[1])",
            "stencils_per_gpu": int(n), "kinds_ee_eep_pe_pep_pp_ppp_pt": [int(k) for k in kinds],
            "outputs": "energy + grad + dense PSD Hessian blocks (12x12/9x9/6x6 families)",
            "parallelism": f"{world} independent replica(s), no collective",
            "l2": "each step writes %.2f GB >> 126 MB L2; no flush needed" % (alg_bytes / 1e9)}


# ---------------------------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port; the Python reference cannot travel)
# ---------------------------------------------------------------------------------------------

def cpu_stencil_baseline(table_np, positions, d_hat, kappa, budget_s, max_rows):
    """C restatement of the reference path, all host threads, on a bounded strided sample."""
    from oracle import c_oracle

    n = len(table_np["kind"])
    stride = max(1, n // max_rows)
    rows = np.arange(0, n, stride)
    sub = {k: np.ascontiguousarray(table_np[k][rows]) for k in ("kind", "verts", "sub", "eps_x")}
    koff = np.searchsorted(sub["kind"], np.arange(8)).astype(np.int64)
    cores = os.cpu_count() or 1
    c_oracle.set_threads(cores)
    prm = c_oracle.make_params(d_hat, kappa)
    out = c_oracle.barrier_stencils(prm, positions, koff, sub["verts"], sub["sub"], sub["eps_x"])  # warm + first touch
    reps, t0 = 0, time.perf_counter()
    while True:
        c_oracle.barrier_stencils(prm, positions, koff, sub["verts"], sub["sub"], sub["eps_x"], out=out)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or reps >= 5000:
            break
    return {"value": len(rows) * reps / el, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{len(rows)} stencils (every {stride}th row of the workload table) x {reps} passes, "
                      f"{el:.1f} s wall; oracle/oracle_c.c with {cores} pthreads, dense block outputs in host RAM"}


def host_table(qb):
    """Contact table of a query batch on the CPU (oracle narrow phase) -- reference arm only."""
    from oracle import tetipc_oracle as o

    return o.narrow_phase(qb.positions, qb.rest_positions, qb.vt, qb.ee, qb.d_hat)


def reference_newton(scene, tab, budget_iters=12):
    """Second half of the metric the way the REFERENCE computes it, on the host, for one scene:
    blocks (assemble_local_quadratics' barrier loop, solver.py:190-216 -- C port, all threads) ->
    group_blocks -> matvec_matrix_free (solver.py:251-262) through the reference's own compiled
    ``kernels._core.matvec_blocks`` (oracle/_ref; single thread, as the reference runs it) -> gradient
    (:218-226) -> block-Jacobi (:265-276) -> ``budget_iters`` iterations of pcg_solve (:279-315).
    The reference has no assembled matrix: its "assembly" is the grouped block list."""
    from oracle import c_oracle
    from oracle import tetipc_oracle as o

    cores = os.cpu_count() or 1
    c_oracle.set_threads(cores)
    koff = np.searchsorted(tab["kind"], np.arange(8)).astype(np.int64)
    prm = c_oracle.make_params(scene.d_hat, scene.kappa, dt=scene.dt)
    args_ = (prm, scene.positions, koff, tab["verts"], tab["sub"], tab["eps_x"])
    out = c_oracle.barrier_stencils(*args_)
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        c_oracle.barrier_stencils(*args_, out=out)
    ms_blocks = (time.perf_counter() - t0) * 1e3 / reps
    verts = tab["verts"]
    fam_rows = {2: np.arange(koff[4], koff[5]), 3: np.arange(koff[2], koff[3]),
                4: np.concatenate([np.arange(koff[k], koff[k + 1]) for k in (0, 1, 3, 5, 6)])}
    grouped, grads = [], []
    for s_ in (2, 3, 4):
        if len(fam_rows[s_]):
            grouped.append((out[f"hess{s_}"], np.ascontiguousarray(verts[fam_rows[s_], :s_].astype(np.int64))))
            grads.append((None, None, grouped[-1][1], out[f"grad{s_}"], None))
    core = c_oracle.reference_core()
    kernel = core.matvec_blocks if core is not None else c_oracle.matvec_blocks
    n = scene.masses.shape[0]
    fixed = np.asarray(scene.fixed, dtype=bool)

    def matvec(v):
        vin = v.copy()
        vin.reshape(n, 3)[fixed] = 0.0
        acc = (scene.masses[:, None] * vin.reshape(n, 3)).reshape(-1).copy()
        for hess, vids in grouped:
            kernel(hess, vids, vin, acc)
        acc.reshape(n, 3)[fixed] = v.reshape(n, 3)[fixed]
        return acc

    v = np.random.default_rng(0).normal(size=3 * n)
    matvec(v)
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        matvec(v)
    ms_matvec = (time.perf_counter() - t0) * 1e3 / reps
    x_tilde = scene.positions + 1e-4 * np.random.default_rng(1).normal(size=scene.positions.shape)
    t0 = time.perf_counter()
    g = o.scatter_gradient(scene.masses, fixed, scene.positions, x_tilde, grads)
    ms_grad = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    o.block_jacobi(grouped, scene.masses, fixed)
    ms_prec = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    _, iters, ok = o.pcg_solve(grouped, scene.masses, fixed, -g, 1e-4, budget_iters, matvec=matvec)
    ms_pcg = (time.perf_counter() - t0) * 1e3 - ms_prec   # pcg_solve rebuilds the preconditioner, like the reference
    per_iter = ms_pcg / max(iters, 1)
    # the reference's OWN pcg_solve (solver.py:279-315, its compiled matvec_blocks) to
    # convergence on the same system -- wall time and iteration count -- when the package is importable
    ref_solve = None
    path = _reference_package_path()
    if path is not None:
        try:
            if path not in sys.path:
                sys.path.insert(0, path)
            import tetipc.kernels as tk
            from tetipc.solver import pcg_solve as ref_pcg_solve

            t0 = time.perf_counter()
            _, it_ref, ok_ref = ref_pcg_solve(grouped, scene.masses, fixed, -g, 1e-4, 2000)
            ref_solve = {"ms": (time.perf_counter() - t0) * 1e3, "iters": int(it_ref), "converged": bool(ok_ref),
                         "backend": tk.BACKEND, "note": "tetipc.solver.pcg_solve, unmodified, one process"}
        except Exception as exc:
            ref_solve = {"error": repr(exc)}
    return {"workload": scene.name, "vertices": int(n), "contacts": int(len(tab["kind"])),
            "reference_pcg_solve": ref_solve,
            "blocks_ms": ms_blocks, "matvec_ms": ms_matvec, "assembly_plus_spmv_ms": ms_blocks + ms_matvec,
            "gradient_ms": ms_grad, "preconditioner_ms": ms_prec, "pcg_ms_per_iter": per_iter,
            "pcg_iters_run": int(iters), "pcg_converged_within_budget": bool(ok),
            "cores": {"blocks": cores, "matvec_pcg": 1},
            "kind": {"blocks": "port (oracle/oracle_c.c)",
                     "matvec": "reference (tetipc.kernels._core.matvec_blocks, oracle/_ref)" if core is not None
                     else "port (oracle_c matvec_blocks)", "pcg": "port of solver.py:279-315 (NumPy) around that matvec"},
            "note": "the reference keeps no assembled matrix: assembly = building the grouped dense block list; "
                    f"PCG bounded to {budget_iters} iterations, per-iteration cost is iteration-independent"}


def host_scene_table(scene):
    """Contact table of a cloth scene on the CPU: host grid broad phase + oracle narrow phase."""
    from oracle import tetipc_oracle as o
    from paper_2308_09400_b200 import workloads

    vt, ee = workloads.broad_phase(scene)
    return o.narrow_phase(scene.positions, scene.rest_positions, vt, ee, scene.d_hat)


def _reference_package_path():
    """Where the UNMODIFIED reference package can be imported from on this box: baseline/_ref (pip-installed by
    __graft_entry__.build(), travels to the GPU box) or the read-only mount of the build container."""
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "tetipc")):
            return path
    return None


def _reference_python_worker(job):
    """One host process of the real-reference arm: the barrier loop of the reference's own
    ``SimState.assemble_local_quadratics`` (solver.py:202-209 -> ``_barrier_block`` :177-184) over its chunk of
    the table, through the reference's own functions, ``reps`` times.  Returns (seconds, blocks built)."""
    path, kind, verts, sub, eps_x, positions, d_hat, kappa, dt, reps = job
    if path not in sys.path:
        sys.path.insert(0, path)
    import tetipc  # noqa: F401
    from tetipc.barrier import BarrierParams, build_local_quadratic
    from tetipc.gap import build_diagonal_jacobian
    from tetipc.mollifier import build_mollified_local_quadratic
    from tetipc.proximity import PARALLEL_KINDS, stencil_distance
    from tetipc.proximity import ContactStencil, StencilKind

    # table rows -> the reference's own ContactStencil objects (kind code = rank of the enum's value string; two bits
    # per local index in `sub`); nothing of this repository is imported in the worker
    order = sorted(StencilKind, key=lambda k: k.value)
    size, sublen = (4, 4, 3, 4, 2, 4, 4), (0, 4, 0, 3, 0, 2, 0)
    stencils = []
    for i in range(len(kind)):
        code = int(kind[i])
        vs = tuple(int(v) for v in verts[i, :size[code]])
        if sublen[code]:
            sel = tuple((int(sub[i]) >> (2 * k)) & 3 for k in range(sublen[code]))
            stencils.append(ContactStencil(kind=order[code], verts=vs, eps_x=float(eps_x[i]), edge_pair=(vs[:2], vs[2:]),
                                           sub=sel, origin=None))
        else:
            stencils.append(ContactStencil(kind=order[code], verts=vs))
    params = BarrierParams(d_hat=d_hat, kappa=kappa)
    dt2, dhat2 = dt * dt, d_hat * d_hat
    built = 0
    t0 = time.perf_counter()
    for _ in range(reps):
        for st in stencils:
            if stencil_distance(st, positions).d2 >= dhat2:      # solver.py:203-205
                continue
            jac = build_diagonal_jacobian(st, positions, d_hat)
            blk = (build_mollified_local_quadratic if st.kind in PARALLEL_KINDS else build_local_quadratic)(st, jac, params)
            blk.grad *= dt2                                         # solver.py:207-208
            blk.hess *= dt2
            built += 1
    return time.perf_counter() - t0, built


class ReferencePython:
    """The reference's own (pure-Python, single-threaded) per-stencil path fanned out over every host core on a
    strided sample of the table; None when the package is not importable on this box."""

    def __init__(self, tab, qb, cores, sample_rows):
        self.path = _reference_package_path()
        self.cores = cores
        n = len(tab["kind"])
        rows = np.unique(np.linspace(0, n - 1, min(sample_rows, n)).astype(np.int64))
        self.n = len(rows)
        chunks = np.array_split(rows, cores)
        # a chunk keeps the table's kind order (rows ascend), so each is a valid kind-sorted table
        self.jobs = []
        for c in chunks:
            if not len(c):
                continue
            verts = tab["verts"][c]
            used, local = np.unique(verts[verts >= 0], return_inverse=True)   # ship only the vertices the chunk touches
            lv = np.full(verts.shape, -1, dtype=verts.dtype)
            lv[verts >= 0] = local
            self.jobs.append((self.path, tab["kind"][c], lv, tab["sub"][c], tab["eps_x"][c],
                              np.ascontiguousarray(qb.positions[used]), float(qb.d_hat), float(qb.kappa), 1.0, 1))
        self.pool = None

    def available(self):
        return self.path is not None

    def __enter__(self):
        import multiprocessing as mp

        # spawn, not fork: the B200 arm calls this with a CUDA context alive in the parent
        self.pool = mp.get_context("spawn").Pool(len(self.jobs))
        return self

    def __exit__(self, *exc):
        self.pool.close()
        self.pool.join()

    def step(self):
        """One pass over the sample on all cores; returns wall seconds.  ``self.per_process`` keeps the rate each
        worker saw for its own chunk (stencils/s of ONE reference process, the reference being single-threaded)."""
        t0 = time.perf_counter()
        res = self.pool.map(_reference_python_worker, self.jobs)
        el = time.perf_counter() - t0
        self.per_process = [len(job[1]) / sec for job, (sec, _) in zip(self.jobs, res)]
        return el


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2308_09400_b200 import workloads

    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    qb = workloads.config2_batch(n=args.n_stencils, seed=20240818)     # rank 0's replica of the B200 arm
    tab = host_table(qb)
    from oracle import c_oracle

    cores = os.cpu_count() or 1
    c_oracle.set_threads(cores)
    koff = np.searchsorted(tab["kind"], np.arange(8)).astype(np.int64)
    prm = c_oracle.make_params(qb.d_hat, qb.kappa)
    out = c_oracle.barrier_stencils(prm, qb.positions, koff, tab["verts"], tab["sub"], tab["eps_x"])

    def step():
        c_oracle.barrier_stencils(prm, qb.positions, koff, tab["verts"], tab["sub"], tab["eps_x"], out=out)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    n = len(tab["kind"])
    port_value = n * args.steps / el
    port = {"value": port_value, "unit": UNIT, "cores": cores, "kind": "port", "ms_per_step": el / args.steps * 1e3,
            "sample": (f"the whole workload table: {n} stencils per step, {args.steps} steps; oracle/oracle_c.c, a C port "
                       f"of the reference's per-stencil path, {cores} pthreads writing the dense block families to host RAM")}
    del out
    # The reference's OWN implementation of the path: the pure-Python barrier loop of assemble_local_quadratics,
    # unmodified, from the installed package (baseline/_ref), one process per host core.  It is the headline value
    # of this arm when the package is importable; the C port above (~300 x faster than it) is reported next to it.
    value, ms_step, baseline = port_value, port["ms_per_step"], dict(port)
    # sample sized so that K steps of it take about a minute at ~10 k stencils/s per core, whatever K is
    ref_py = ReferencePython(tab, qb, cores, sample_rows=min(100_000, max(8_000, int(60 * 10_000 * cores / (args.steps + 1)))))
    if ref_py.available():
        with ref_py:
            for _ in range(min(args.warmup, 1)):
                ref_py.step()
            secs = [ref_py.step() for _ in range(args.steps)]
        value = ref_py.n * args.steps / sum(secs)
        ms_step = sum(secs) / args.steps * 1e3
        baseline = {"value": value, "unit": UNIT, "cores": len(ref_py.jobs), "kind": "reference",
                    "one_process": float(np.median(ref_py.per_process)),
                    "sample": (f"{ref_py.n} stencils per step (every {n // max(ref_py.n, 1)}th row of the {n}-row workload table, "
                               f"all kinds in proportion), {args.steps} steps; the unmodified tetipc package from "
                               f"{os.path.relpath(ref_py.path, ROOT) if ref_py.path.startswith(ROOT) else ref_py.path}: "
                               f"stencil_distance -> build_diagonal_jacobian -> build_(mollified_)local_quadratic per stencil "
                               f"(solver.py:177-209), {len(ref_py.jobs)} processes (the reference itself is single-threaded)")}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(n, np.diff(koff), world, algorithmic_bytes(koff, qb.positions.shape[0])),
        "cpu_baseline": baseline,
        "c_port": port,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    # the vectorised NumPy oracle (one process) and the reference's own
    # `bench-projection` command, for continuity with PAPER.md:784-802
    try:
        from oracle import tetipc_oracle as o_

        rows = np.arange(0, n, max(1, n // 250_000))
        t0 = time.perf_counter()
        o_.local_quadratics_batch(tab["kind"][rows], tab["verts"][rows], tab["sub"][rows], tab["eps_x"][rows], qb.positions,
                                  qb.d_hat, qb.kappa)
        line["numpy_oracle"] = {"value": len(rows) / (time.perf_counter() - t0), "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"{len(rows)} stencils, oracle/tetipc_oracle.py local_quadratics_batch, one process"}
    except Exception as exc:
        line["numpy_oracle"] = {"error": repr(exc)}
    path = _reference_package_path()
    if path is not None and not args.skip_newton:    # the long legs ride with the full run only
        import subprocess

        proj = {}
        for count in (100_000, 1_000_000):
            try:
                outp = subprocess.run([sys.executable, "-m", "tetipc.cli", "bench-projection", "--count", str(count), "--dim", "12"],
                                      capture_output=True, text=True, timeout=300, env=dict(os.environ, PYTHONPATH=path),
                                      cwd="/tmp").stdout.strip().splitlines()[-1]
                proj[str(count)] = json.loads(outp)
            except Exception as exc:
                proj[str(count)] = {"error": repr(exc)}
        line["reference_bench_projection"] = proj
    if not args.skip_newton:
        line["newton"] = {}
        for key, scene in (("cloth_stack", workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)),
                           ("cloth_on_sphere", workloads.cloth_on_sphere())):
            try:
                line["newton"][key] = reference_newton(scene, host_scene_table(scene))
            except Exception as exc:  # the headline above stands on its own
                line["newton"][key] = {"error": repr(exc)}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------------------------

def newton_section(torch, pkg, steps, warmup, peak, cloth, extras=True, cpu_leg=True):
    """Assembly + SpMV (+ PCG) on one cloth scene: BASELINE configs[3] (teaser-style stack, ~1M contacts;
    ``extras``: CCD, friction, elasticity, whole time steps) or configs[2] (cloth on sphere, ~100k vertices)."""
    workloads, contacts, stencils, solver, barrier, device, _lib = pkg
    params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
    pos = device.to_device(cloth.positions)
    d_rest = device.to_device(cloth.rest_positions)
    # detect = broad phase (grid join) + narrow phase (classify, filter, promote, sort), all on the device
    bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
    d_vt, d_ee = bp.query(pos)  # warm (module load, workspace allocation)
    contacts.narrow_phase_device(pos, d_rest, d_vt, d_ee, cloth.d_hat, want_origin=False)
    def wall_ms(fn, reps=5):
        """Best of `reps` wall-clock runs bracketed by synchronize (host-synchronising entry points)."""
        best, out = float("inf"), None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) * 1e3)
        return best, out

    ms_broad, (d_vt, d_ee) = wall_ms(lambda: bp.query(pos))
    ms_narrow, (table, extra_np) = wall_ms(lambda: contacts.narrow_phase_device(pos, d_rest, d_vt, d_ee, cloth.d_hat,
                                                                                want_origin=False))
    t_broad, t_narrow = ms_broad * 1e-3, ms_narrow * 1e-3
    n_queries = int(d_vt.shape[0]) + int(d_ee.shape[0])
    batch = stencils.evaluate(table, pos, params, dt=cloth.dt, want_factors=True)
    batch.raise_on_penetration()
    fams = [batch.families[s] for s in sorted(batch.families)]
    sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
    ms_stencil = time_steps(torch, lambda: stencils.evaluate(table, pos, params, dt=cloth.dt, out=batch), steps, warmup) / steps
    sysm.set_pattern([(f.s, f.vids) for f in fams])  # warm (module load, workspace allocation)
    ms_symbolic, nnzb = wall_ms(lambda: sysm.set_pattern([(f.s, f.vids) for f in fams]), reps=3)
    hess = [f.hess for f in fams]
    ms_numeric = time_steps(torch, lambda: sysm.assemble(hess), steps, warmup) / steps
    sysm.set_numeric_variant(4)
    ms_numeric_rows = time_steps(torch, lambda: sysm.assemble(hess), steps, warmup) / steps
    sysm.set_numeric_variant(0)
    # fused path: the matrix straight from the rank-1 factors, dense blocks never materialised
    fac = [f.fac for f in fams]
    ms_factors = time_steps(torch, lambda: sysm.assemble_from_factors(fac), steps, warmup) / steps
    lean = stencils.evaluate(table, pos, params, dt=cloth.dt, want_hess=False, want_factors=True)
    ms_stencil_lean = time_steps(torch, lambda: stencils.evaluate(table, pos, params, dt=cloth.dt, want_hess=False,
                                                                   want_factors=True, out=lean), steps, warmup) / steps
    del lean
    sysm.assemble(hess)
    x = device.to_device(np.random.default_rng(0).normal(size=3 * sysm.n))
    y = device.empty((3 * sysm.n,))
    ms_spmv = time_steps(torch, lambda: sysm.spmv(x, out=y), steps, warmup) / steps
    x_tilde = cloth.positions + 1e-4 * np.random.default_rng(1).normal(size=cloth.positions.shape)
    xt = device.to_device(x_tilde)
    grads = [f.grad for f in fams]
    ms_grad = time_steps(torch, lambda: sysm.gradient(pos, xt, grads), steps, warmup) / steps
    rhs = -sysm.gradient(pos, xt, grads)
    sysm.block_jacobi()
    iters_cap = 50
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d, iters, ok, _, _ = sysm.pcg(rhs, 1e-30, iters_cap)
    t1 = time.perf_counter()
    d, iters2, ok, _, _ = sysm.pcg(rhs, 1e-30, 5 * iters_cap)
    # slope between a 50- and a 250-iteration solve: launch, result copy and sync cancel
    ms_pcg_iter = ((time.perf_counter() - t1) - (t1 - t0)) * 1e3 / max(iters2 - iters, 1)
    t0 = time.perf_counter()
    d, it_full, ok_full, _, _ = sysm.pcg(rhs, 1e-4, 2000)
    ms_pcg_full = (time.perf_counter() - t0) * 1e3
    # the paper's alternative preconditioner: multilevel additive Schwarz, same stopping rule
    sysm.mas_order(pos)
    ms_mas_order, _ = wall_ms(lambda: sysm.mas_order(pos), reps=3)
    mas = {}
    for lv in (1, 2):
        sysm.mas_setup(lv)
        ms_setup, _ = wall_ms(lambda: sysm.mas_setup(lv), reps=3)
        sysm._mas_stale = False
        sysm.pcg(rhs, 1e-4, 2000, preconditioner="mas", mas_levels=lv)
        ms_solve, (_, it_mas, ok_mas, _, _) = wall_ms(lambda: sysm.pcg(rhs, 1e-4, 2000, preconditioner="mas", mas_levels=lv), reps=3)
        mas[f"levels_{lv}"] = {"setup_ms": ms_setup, "solve_ms": ms_solve, "iters": it_mas, "converged": ok_mas,
                               "us_per_iter": ms_solve * 1e3 / max(it_mas, 1), "setup_plus_solve_ms": ms_setup + ms_solve}
    mas["order_ms"] = ms_mas_order
    mas["note"] = ("Morton-ordered 32-vertex domains, fp32 symmetric-half inverses, fused into the persistent PCG kernel; "
                   "stops on the reference's block-Jacobi-norm rule like pcg_solve_ms; setup is paid per Newton iteration "
                   "(the matrix changes), order once per time step")
    if extras:
        # CCD step filter of the line search: swept-AABB candidates + ACCD bound, on the device
        dirs = device.to_device(0.3 * cloth.d_hat * np.random.default_rng(3).normal(size=cloth.positions.shape))
        alpha = bp.ccd_step_bound(pos, dirs)  # warm
        s_vt, s_ee = bp.sweep(pos, dirs)
        ms_ccd, alpha = wall_ms(lambda: bp.ccd_step_bound(pos, dirs), reps=3)
        ms_ccd_filter = time_steps(torch, lambda: contacts.ccd_filter_device(s_vt, s_ee, pos, dirs), 3, 1) / 3
        # friction: lagged state once per time step, blocks once per Newton iteration
        from paper_2308_09400_b200 import friction as friction_mod

        raw = stencils.evaluate(table, pos, params, dt=1.0, want_energy=False, want_hess=False)
        fstate = friction_mod.update_state(table, pos, 0.4, 1e-3, cloth.dt, barrier_batch=raw)  # warm
        ms_fstate, fstate = wall_ms(lambda: friction_mod.update_state(table, pos, 0.4, 1e-3, cloth.dt, barrier_batch=raw), reps=3)
        x_moved = device.to_device(cloth.positions + 0.5 * cloth.dt * 1e-3 * np.random.default_rng(4).normal(size=cloth.positions.shape))
        friction_mod.evaluate(fstate, x_moved, pos)
        ms_fblocks = time_steps(torch, lambda: friction_mod.evaluate(fstate, x_moved, pos), 10, 2) / 10
        fr_bytes = sum(int(fstate.table.family_count(s_)) * (72 * s_ * s_ + 24 * s_ + 4 * s_ + 96) for s_ in (2, 3, 4))
        del raw
        # elasticity: 400k random tets, energy + gradient + analytically projected 12x12 block each
        from paper_2308_09400_b200 import elasticity as elasticity_mod

        rng_e = np.random.default_rng(11)
        n_tet = 400_000
        rest_t = rng_e.normal(size=(4 * n_tet, 3))
        tets_t = np.arange(4 * n_tet).reshape(n_tet, 4)
        mesh_t = elasticity_mod.TetMesh(rest_t, tets_t, 3.7e4, 8.6e4)
        x_t = device.to_device(rest_t + 0.1 * rng_e.normal(size=rest_t.shape))
        mesh_t.evaluate(x_t, dt=cloth.dt)
        ms_elastic = time_steps(torch, lambda: mesh_t.evaluate(x_t, dt=cloth.dt), 5, 1) / 5
        del mesh_t, x_t
    # one whole Newton direction through the public device-resident API, host arrays in, host array out:
    # H2D (x, x~) -> detect -> stencils (factors) -> symbolic + numeric assembly -> gradient -> PCG -> D2H d
    x_host = np.ascontiguousarray(cloth.positions)
    xt_host = np.ascontiguousarray(x_tilde)

    def newton_direction(prec="block_jacobi"):
        px, pxt = device.to_device(x_host), device.to_device(xt_host)
        cvt, cee = bp.query(px)
        tab, _ = contacts.narrow_phase_device(px, d_rest, cvt, cee, cloth.d_hat, want_origin=False)
        b = stencils.evaluate(tab, px, params, dt=cloth.dt, want_hess=False, want_factors=True)
        fl = [b.families[s_] for s_ in sorted(b.families)]
        sysm.set_pattern([(f.s, f.vids) for f in fl])
        sysm.assemble_from_factors([f.fac for f in fl])
        g = sysm.gradient(px, pxt, [f.grad for f in fl])
        sysm.block_jacobi()
        if prec == "mas":
            sysm.mas_order(px)
        dd, its, okk, _, _ = sysm.pcg(-g, 1e-4, 2000, preconditioner=prec)
        return device.to_host(dd), its, okk, float(b.summary()[0])

    e2e = {}
    for prec in ("block_jacobi", "mas"):
        for _ in range(2):   # the second call still pays first-use costs (list regrowth, descriptor tables, allocator)
            newton_direction(prec)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps_e2e = 5
        for _ in range(reps_e2e):
            d_host, its_e2e, ok_e2e, energy_e2e = newton_direction(prec)
        e2e[prec] = ((time.perf_counter() - t0) * 1e3 / reps_e2e, its_e2e, ok_e2e)
    ms_newton_e2e, its_e2e, ok_e2e = e2e["block_jacobi"]
    n_c = table.n
    ent = sum(int(f.vids.shape[0]) * f.s * f.s for f in fams)
    num_bytes = sum(int(f.vids.shape[0]) * (72 * f.s * f.s) for f in fams) + 4 * ent + 72 * nnzb
    spmv_bytes = 76 * nnzb + 52 * sysm.n
    fac_bytes = sum(int(f.vids.shape[0]) * 24 * f.s for f in fams) + 4 * ent + 72 * nnzb
    out = {
        "workload": cloth.name + f" d_hat={cloth.d_hat:.3g}",
        "vertices": sysm.n, "contacts": n_c, "kinds": np.diff(table.kind_off).tolist(), "nnzb": nnzb,
        "candidate_queries": n_queries, "broad_phase_ms": t_broad * 1e3, "narrow_phase_ms": t_narrow * 1e3,
        "detect_ms": (t_broad + t_narrow) * 1e3,
        "stencils_ms": ms_stencil, "symbolic_ms": ms_symbolic, "assembly_numeric_ms": ms_numeric, "assembly_numeric_rowwise_ms": ms_numeric_rows, "spmv_ms": ms_spmv,
        "fused": {"stencils_factors_only_ms": ms_stencil_lean, "assembly_from_factors_ms": ms_factors,
                  "note": "rank-1 path: the stencil kernel writes z (24 s bytes) instead of the dense block and the "
                          "assembly gathers from z; same matrix bit for bit"},
        "assembly_plus_spmv_ms": ms_numeric + ms_spmv, "gradient_scatter_ms": ms_grad,
        "per_newton_iteration_ms": {"symbolic": ms_symbolic, "numeric_from_factors": ms_factors, "spmv": ms_spmv,
                                    "total": ms_symbolic + ms_factors + ms_spmv,
                                    "note": "the contact set changes every Newton iteration, so the symbolic phase is "
                                            "paid every time: this is the honest assembly+SpMV figure of the solver loop"},
        "newton_direction_e2e": {"ms": ms_newton_e2e, "pcg_iters": its_e2e, "converged": ok_e2e,
                                 "h2d_bytes": 2 * x_host.nbytes, "d2h_bytes": int(d_host.nbytes) + 8,
                                 "note": "host x, x~ in -> detect, stencils (rank-1 factors), symbolic + numeric assembly, "
                                         "gradient, block-Jacobi PCG to 1e-4 -> host direction + energy out; wall clock"},
        "newton_direction_e2e_mas": {"ms": e2e["mas"][0], "pcg_iters": e2e["mas"][1], "converged": e2e["mas"][2],
                                     "note": "the same call with preconditioner='mas' (Morton order + domain inverses "
                                             "rebuilt inside the timed region)"},
        "pcg_ms_per_iter": ms_pcg_iter, "pcg_solve_ms": ms_pcg_full, "pcg_iters": it_full, "pcg_converged": ok_full,
        "pcg_mas": mas,
        "roofline_assembly": {"bound": "hbm", "achieved": num_bytes / ms_numeric / 1e6, "peak": peak, "unit": "GB/s",
                              "frac": num_bytes / ms_numeric / 1e6 / peak},
        "roofline_assembly_factors": {"bound": "hbm", "achieved": fac_bytes / ms_factors / 1e6, "peak": peak,
                                      "unit": "GB/s", "frac": fac_bytes / ms_factors / 1e6 / peak,
                                      "algorithmic_bytes": fac_bytes},
        "roofline_spmv": {"bound": "hbm", "achieved": spmv_bytes / ms_spmv / 1e6, "peak": peak, "unit": "GB/s",
                          "frac": spmv_bytes / ms_spmv / 1e6 / peak},
    }
    if extras:
        out["ccd"] = {"sweep_candidates": int(s_vt.shape[0]) + int(s_ee.shape[0]), "sweep_plus_filter_ms": ms_ccd,
                      "filter_kernel_ms": ms_ccd_filter, "alpha": alpha, "note": "sweep_candidates + global_ccd_filter (proximity.py:388-432), random 0.3 d_hat step"}
        out["friction"] = {"data": int(fstate.n), "state_ms": ms_fstate, "blocks_ms": ms_fblocks,
                           "blocks_GBps": fr_bytes / ms_fblocks / 1e6,
                           "note": "update_friction_state (once per time step) and friction energy/grad/rank-2 PSD blocks "
                                   "(once per Newton iteration, incl. output allocation) on the same contact table"}
        out["elastic"] = {"tets": n_tet, "blocks_ms": ms_elastic, "tets_per_s": n_tet / ms_elastic * 1e3,
                          "note": "stable neo-Hookean energy + gradient + analytically PSD-projected 12x12 per tet (incl. output allocation)"}
    # CPU side of the same half of the metric, on the same contact table: the reference's way of doing it
    # (blocks -> grouped list -> compiled matvec_blocks inside its PCG recurrence), bounded
    if cpu_leg:
        try:
            tab_np = {"kind": device.to_host(extra_np.kind), "verts": device.to_host(table.verts),
                      "sub": device.to_host(table.sub), "eps_x": device.to_host(table.eps_x)}
            ref = reference_newton(cloth, tab_np)
            out["reference_cpu"] = ref
            out["vs_reference_cpu"] = {
                "assembly_plus_spmv": ref["assembly_plus_spmv_ms"] / (ms_numeric + ms_spmv),
                "pcg_per_iter": ref["pcg_ms_per_iter"] / ms_pcg_iter,
                "newton_direction": (ref["blocks_ms"] + ref["gradient_ms"] + ref["preconditioner_ms"]
                                     + it_full * ref["pcg_ms_per_iter"]) / ms_newton_e2e,
                "pcg_solve": (ref["reference_pcg_solve"]["ms"] / ms_pcg_full
                              if ref.get("reference_pcg_solve") and "ms" in ref["reference_pcg_solve"] else None),
                "pcg_solve_vs_mas": (ref["reference_pcg_solve"]["ms"] / mas["levels_1"]["setup_plus_solve_ms"]
                                     if ref.get("reference_pcg_solve") and "ms" in ref["reference_pcg_solve"] else None),
                "pcg_iters_reference_vs_here": ([ref["reference_pcg_solve"].get("iters"), it_full]
                                                if ref.get("reference_pcg_solve") else None),
                "note": "reference-side time / B200 time; pcg_solve = the unmodified tetipc.solver.pcg_solve to 1e-4 on the "
                        "same system against NewtonSystem.pcg (block-Jacobi) and against MAS setup + solve; "
                        "the reference's Newton direction is projected as blocks + "
                        "gradient + preconditioner + (this solve's iteration count) x its measured per-iteration cost, "
                        "detect excluded on the reference side and included on the B200 side"}
            if extras:  # the reference's own compiled ACCD on a sample of the swept candidates
                from oracle import c_oracle

                core = c_oracle.reference_core()
                if core is not None:
                    xs, ds = device.to_host(pos), device.to_host(dirs)
                    cand = device.to_host(s_vt[:20000]).astype(np.int64)
                    t0 = time.perf_counter()
                    for row in cand:
                        core.accd_max_step(xs[row], ds[row], 0, 0.9)
                    out["ccd"]["cpu_pairs_per_s"] = len(cand) / (time.perf_counter() - t0)
                    out["ccd"]["cpu_kind"] = "reference (tetipc.kernels._core.accd_max_step, 1 core, Python call per pair)"
        except Exception as exc:  # baseline only; never fail the bench on it
            out["reference_cpu"] = {"error": repr(exc)}
    sysm.close()
    bp.close()
    if not extras:
        return out
    # whole time steps through the stepper (the reference's advance_time_step on the device path): a softer
    # cloth stack of the same size whose Newton loop converges (the stiff one above is a kernel workload)
    from paper_2308_09400_b200 import stepper

    soft = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2, jitter_rel=0.01, kappa=1e5)
    cfg = stepper.SolverConfig(dt=soft.dt, barrier=barrier.BarrierParams(d_hat=soft.d_hat, kappa=soft.kappa))
    # the same three steps twice, the second pass reported: the first one pays every first use (lazily loaded
    # kernels, list and workspace growth: 370 - 450 ms for the first step of a fresh process against 127 ms)
    for timed in (False, True):
        state = stepper.SimState(soft.as_scene(), cfg)
        steps_out = []
        for _ in range(3):
            n_start = state.detect(state.x).n
            st = stepper.advance_time_step(state)
            steps_out.append({"contacts_at_start": n_start, "newton_iters": st.newton_iters, "pcg_iters": st.pcg_iters,
                              "converged": st.converged, "min_distance_over_d_hat": st.min_distance / soft.d_hat,
                              "wall_ms": st.wall_ms})
        state.close()
    out["time_step"] = {"workload": soft.name + " kappa=1e5 jitter=0.01h (shells, no membrane energy)",
                        "vertices": state.n, "steps": steps_out,
                        "note": "stepper.advance_time_step: detect, blocks, assembly, PCG, CCD, line search (re-detect "
                                "per candidate), end-of-step detect; wall clock incl. every host sync; second of two "
                                "passes over the same three steps (the first pass pays the first-use costs)"}
    return out


def run_dry(args):
    """CPU rehearsal of the N-rank path (launch, rank environment, timed bracket, aggregate) with gloo: a step
    is the generation of the rank's own replica workload.  Prints a line flagged ``dry_run``; never a bench value."""
    from paper_2308_09400_b200 import scene_batch, workloads

    rank, world, _, dist = scene_batch.init(backend="gloo")
    seed = scene_batch.replica_seed(20240818, rank)
    state = {}

    def step():
        state["qb"] = workloads.config2_batch(n=2000, seed=seed)

    ms = scene_batch.timed_steps(step, args.steps, args.warmup, dist, cuda=False)
    units, ms_max = scene_batch.aggregate(len(state["qb"].ee), ms, dist)
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": "replica workloads generated/s (CPU rehearsal, not a bench value)",
                          "value": scene_batch.throughput(units, ms_max, args.steps), "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "units_per_step_all_ranks": units,
                          "ms_per_step": ms_max / args.steps, "scaling": "weak"}), flush=True)
    scene_batch.finish(dist)


def run_b200(args):
    import torch

    from paper_2308_09400_b200 import scene_batch

    rank, world, local, dist = scene_batch.init(backend="nccl")

    def barrier():
        scene_batch.barrier(dist)

    from paper_2308_09400_b200 import _lib, barrier as barrier_mod, contacts, device, solver, stencils, workloads

    L = _lib.lib()
    peak, peak_src = measured_peak()

    # ---- workload: config 2, one independent replica per rank ----------------------------------
    qb = workloads.config2_batch(n=args.n_stencils, seed=scene_batch.replica_seed(20240818, rank))
    params = barrier_mod.BarrierParams(d_hat=qb.d_hat, kappa=qb.kappa)
    pos = device.to_device(qb.positions)
    table, extra = contacts.narrow_phase_device(pos, qb.rest_positions, qb.vt, qb.ee, qb.d_hat, want_origin=False)
    n = table.n
    batch = stencils.evaluate(table, pos, params)
    batch.raise_on_penetration()
    alg_bytes = algorithmic_bytes(table.kind_off, pos.shape[0])

    def step():
        stencils.evaluate(table, pos, params, out=batch)

    launches0 = L.b200ipc_launch_count()
    clocks = ClockSampler(local)
    clocks.__enter__()  # sampled across the device-timed and the end-to-end regions below
    ms_total = time_steps(torch, step, args.steps, args.warmup, dist)
    # counted by the library: launches of (warm-up + timed) steps, scaled to the timed region
    counted = int(L.b200ipc_launch_count() - launches0)
    per_step_launches = counted // (args.steps + args.warmup)
    assert per_step_launches == 1, (counted, args.steps, args.warmup)  # one fused launch per step
    gpu_launches = per_step_launches * args.steps

    total_stencils, ms_max = scene_batch.aggregate(n, ms_total, dist, device="cuda")
    ms_per_step = ms_max / args.steps
    value = scene_batch.throughput(total_stencils, ms_max, args.steps)

    # ---- end to end through the public API with HOST buffers ------------------------------------
    # strict: pinned host inputs -> H2D -> kernel -> every output (energy, status, grad, hess) D2H
    h_pos = torch.from_numpy(qb.positions).pin_memory()
    h_verts = table.verts.cpu().pin_memory()
    h_sub = table.sub.cpu().pin_memory()
    h_eps = table.eps_x.cpu().pin_memory()
    outs = [batch.energy, batch.status] + [t_ for f in batch.families.values() for t_ in (f.grad, f.hess)]
    h_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs]
    h2d = h_pos.numel() * 8 + h_verts.numel() * 4 + h_sub.numel() + h_eps.numel() * 8
    d2h = sum(o.numel() * o.element_size() for o in outs)

    # Double-buffered device outputs and a second stream: the D2H of step k runs on the copy stream while
    # the H2D and the kernel of step k+1 run on the compute stream (PCIe is full duplex).  Every step still
    # moves all of its inputs H2D and all of its outputs D2H inside the timed region.
    batch_b = stencils.evaluate(table, pos, params)
    bufs = [batch, batch_b]
    outs_of = [[b.energy, b.status] + [t_ for f in b.families.values() for t_ in (f.grad, f.hess)] for b in bufs]
    copy_stream = torch.cuda.Stream()
    drained = [torch.cuda.Event(), torch.cuda.Event()]
    for ev in drained:
        ev.record()

    def e2e_step(full, k):
        cur = torch.cuda.current_stream()
        b = bufs[k % 2]
        d_pos = h_pos.cuda(non_blocking=True)
        tab = stencils.DeviceStencilTable(n, table.kind_off, h_verts.cuda(non_blocking=True),
                                          h_sub.cuda(non_blocking=True), h_eps.cuda(non_blocking=True))
        if full:
            cur.wait_event(drained[k % 2])          # the copy that last read this output buffer is done
        stencils.evaluate(tab, d_pos, params, out=b)
        if full:
            copy_stream.wait_stream(cur)
            with torch.cuda.stream(copy_stream):
                for o, h in zip(outs_of[k % 2], h_out):
                    h.copy_(o, non_blocking=True)
                    o.record_stream(copy_stream)
                drained[k % 2].record(copy_stream)
        else:
            b._summary = None
            b.summary()  # device reduction + D2H of (energy sum, inactive, penetrating)

    def time_e2e(full, steps_, warm_):
        cur = torch.cuda.current_stream()
        for k in range(warm_):
            e2e_step(full, k)
        cur.wait_stream(copy_stream)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(steps_):
            e2e_step(full, k)
        cur.wait_stream(copy_stream)               # the last step's outputs are on the host before the clock stops
        e1.record()
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1)

    e2e_steps = max(4, min(args.steps, 10))
    ms_e2e = time_e2e(True, e2e_steps, 2) / e2e_steps
    ms_res = time_e2e(False, e2e_steps, 2) / e2e_steps
    del batch_b, bufs, outs_of
    te = torch.tensor([ms_e2e, ms_res], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    ms_e2e, ms_res = float(te[0].item()), float(te[1].item())
    del h_out
    clocks.__exit__(None, None, None)

    line = None
    if rank == 0:
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "stencil_traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as fh:
                tj = json.load(fh)
            if tj.get("stencils") == n:
                traffic = tj.get("dram_bytes_per_step")
        achieved = alg_bytes / (ms_total / args.steps) / 1e6  # rank 0's own kernel time
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(n, np.diff(table.kind_off), world, alg_bytes),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "peak_source": peak_src,
                         "kernel": "barrier_stencil_kernel (one fused launch per step, CTA-uniform kind dispatch)",
                         "algorithmic_bytes_per_step": alg_bytes},
            "e2e": {"value": total_stencils / (ms_e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
                    "note": "pinned host inputs -> H2D -> kernel -> every output D2H into pinned host memory, double-buffered: the D2H of step k overlaps the H2D + kernel of step k+1 (PCIe bound)",
                    "resident_value": total_stencils / (ms_res * 1e-3), "resident_ms_per_step": ms_res,
                    "resident_d2h_bytes_per_step": 24,
                    "resident_note": "same H2D; blocks stay in HBM for the on-device assembly/PCG, only the energy "
                                     "sum and status counts return"},
            "gpu_launches": gpu_launches,
            "clocks": clocks.summary(),
        }
    # ---- second half of the metric + CPU baseline: rank 0, single-GPU runs only -------------------
    pkg = (workloads, contacts, stencils, solver, barrier_mod, device, _lib)
    if rank == 0 and world == 1 and not args.skip_newton:
        del batch
        torch.cuda.empty_cache()
        stack = workloads.cloth_stack(layers=4, n=140, seed=1, d_hat_rel=0.2)
        line["newton"] = newton_section(torch, pkg, 20, 3, peak, stack, extras=True, cpu_leg=not args.skip_cpu)
        torch.cuda.empty_cache()
        line["newton_cloth_on_sphere"] = newton_section(torch, pkg, 20, 3, peak, workloads.cloth_on_sphere(),
                                                        extras=False, cpu_leg=not args.skip_cpu)
        line["fp64"] = fp64_section(torch, L, line)
    if rank == 0 and world == 1 and not args.skip_cpu:
        tab_np = {"kind": device.to_host(extra.kind), "verts": device.to_host(table.verts),
                  "sub": device.to_host(table.sub), "eps_x": device.to_host(table.eps_x)}
        try:
            line["cpu_baseline"] = cpu_stencil_baseline(tab_np, qb.positions, qb.d_hat, qb.kappa, 12.0, 250_000)
        except Exception as exc:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"unavailable: {exc}"}
        # and the reference's own pure-Python path (what `--impl reference` reports), on a small sample
        try:
            ref_py = ReferencePython(tab_np, qb, os.cpu_count() or 1, sample_rows=32_000)
            if ref_py.available():
                with ref_py:
                    ref_py.step()
                    sec = ref_py.step()
                line["cpu_reference_python"] = {"value": ref_py.n / sec, "unit": UNIT, "cores": len(ref_py.jobs),
                                                "kind": "reference",
                                                "sample": f"{ref_py.n} stencils, one pass after a warm-up pass, "
                                                          f"{len(ref_py.jobs)} processes of the unmodified tetipc package"}
        except Exception as exc:
            line["cpu_reference_python"] = {"value": None, "kind": "reference", "sample": f"unavailable: {exc}"}
    # ---- BASELINE configs[4]: N independent multilayer-cloth scenes, one per GPU --------------------
    if world > 1 and not args.skip_newton:
        batch = None
        torch.cuda.empty_cache()
        sb = scene_batch_section(torch, pkg, scene_batch, dist, rank, world)
        if rank == 0:
            line["scene_batch"] = sb
    if rank == 0:
        print(json.dumps(line), flush=True)
    scene_batch.finish(dist)


def scene_batch_section(torch, pkg, scene_batch, dist, rank, world, reps=5):
    """configs[4]: every rank owns one teaser-style cloth stack (its own seed) and computes whole Newton
    directions for it, host positions in, host direction out; scenes/s = all ranks' directions over the
    slowest rank's time.  No collective on the data path."""
    workloads, contacts, stencils, solver, barrier, device, _lib = pkg
    cloth = workloads.cloth_stack(layers=4, n=140, seed=scene_batch.replica_seed(1, rank), d_hat_rel=0.2)
    params = barrier.BarrierParams(d_hat=cloth.d_hat, kappa=cloth.kappa)
    d_rest = device.to_device(cloth.rest_positions)
    bp = contacts.BroadPhase(None, cloth.tris, cloth.edges, cloth.d_hat, cloth.positions)
    sysm = solver.NewtonSystem(cloth.masses, cloth.fixed)
    x_host = torch.from_numpy(np.ascontiguousarray(cloth.positions)).pin_memory()
    xt_host = torch.from_numpy(cloth.positions + 1e-4 * np.random.default_rng(1).normal(size=cloth.positions.shape)).pin_memory()
    stats = {}

    def direction():
        px, pxt = x_host.cuda(non_blocking=True), xt_host.cuda(non_blocking=True)
        cvt, cee = bp.query(px)
        tab, _ = contacts.narrow_phase_device(px, d_rest, cvt, cee, cloth.d_hat, want_origin=False)
        b = stencils.evaluate(tab, px, params, dt=cloth.dt, want_hess=False, want_factors=True)
        fl = [b.families[s_] for s_ in sorted(b.families)]
        sysm.set_pattern([(f.s, f.vids) for f in fl])
        sysm.assemble_from_factors([f.fac for f in fl])
        g = sysm.gradient(px, pxt, [f.grad for f in fl])
        sysm.block_jacobi()
        dd, its, okk, _, _ = sysm.pcg(-g, 1e-4, 2000)
        stats.update(contacts=tab.n, pcg_iters=its, converged=bool(okk), d=device.to_host(dd))

    ms = scene_batch.timed_steps(direction, reps, 2, dist, cuda=True)
    scenes, ms_max = scene_batch.aggregate(1.0, ms, dist, device="cuda")
    contacts_total, _ = scene_batch.aggregate(stats["contacts"], ms, dist, device="cuda")
    sysm.close()
    bp.close()
    return {"workload": "BASELINE configs[4]: one cloth-stack-4x140x140 scene per GPU (seed = 1 + rank)",
            "scenes": scenes, "contacts_all_scenes": contacts_total, "newton_direction_ms_slowest_rank": ms_max / reps,
            "scenes_per_s": scene_batch.throughput(scenes, ms_max, reps),
            "contacts_per_s": scene_batch.throughput(contacts_total, ms_max, reps),
            "rank0": {"contacts": stats["contacts"], "pcg_iters": stats["pcg_iters"], "converged": stats["converged"]},
            "note": "host x, x~ in -> detect, stencils, symbolic + numeric assembly, gradient, PCG to 1e-4 -> host "
                    "direction out; barrier + synchronize bracket, max over ranks; weak scaling"}


def fp64_section(torch, L, line):
    """DFMA peak measured on this GPU (b200ipc_fp64_probe) and the fp64 rooflines of the two kernels that are
    not HBM-bound; flop counts from the kernel headers (csrc/accd.cu, csrc/elastic.cu)."""
    import ctypes as C

    tf = C.c_double(0.0)
    rc = L.b200ipc_fp64_probe(C.byref(tf), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    out = {"fp64_tflops_measured": tf.value if rc == 0 else None,
           "how": "b200ipc_fp64_probe: 8 independent DFMA chains per thread, 148 x 32 CTAs x 256 threads, best of 5"}
    # fp64 flops per launch of the two compute-bound kernels: counted by ncu (2 x DFMA + DADD + DMUL thread
    # instructions, profiles/fp64_flops.json, same workloads as timed here); times are this run's
    path = os.path.join(ROOT, "profiles", "fp64_flops.json")
    if rc == 0 and os.path.exists(path):
        with open(path) as fh:
            counted = json.load(fh)
        newton = line.get("newton", {})
        times = {"accd_kernel": newton.get("ccd", {}).get("filter_kernel_ms"),
                 "elastic_blocks_kernel": newton.get("elastic", {}).get("blocks_ms")}
        for name, ms in times.items():
            c = counted.get(name)
            if c and ms:
                ach = c["flops_per_launch"] / (ms * 1e-3) / 1e12
                out["roofline_" + name] = {"bound": "fp64", "achieved": ach, "peak": tf.value, "unit": "TFLOP/s",
                                           "frac": ach / tf.value, "flops_per_launch": c["flops_per_launch"],
                                           "workload": c.get("workload")}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n-stencils", type=int, default=1_000_000)
    ap.add_argument("--skip-newton", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo rehearsal of the N-rank launch + aggregate path")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: become N ranks, one per GPU, exactly as the driver would launch us
        from paper_2308_09400_b200 import scene_batch

        sys.exit(scene_batch.launch(args.gpus, [os.path.abspath(__file__)] + sys.argv[1:]))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
