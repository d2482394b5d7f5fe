"""Assembly, matvec, block-Jacobi and PCG: the reference's solver entry points on the GPU.

Host-array twins keep the reference's names and signatures
(``/root/reference/pkg/src/tetipc/solver.py:237-315``): ``group_blocks``,
``matvec_matrix_free``, ``block_jacobi_preconditioner``, ``pcg_solve``.  ``NewtonSystem`` is
the device-resident object they are built on: it owns the assembled 3x3-block sparse matrix of
one scene and is what a GPU-resident Newton loop uses directly (no host round trips between
stencil evaluation, assembly, gradient and the PCG solve).
"""

import ctypes as C

import numpy as np

from . import _lib, device
from .kernels import matvec_blocks_device


def group_blocks(blocks):
    """Stack ``LocalQuadratic`` blocks by stencil size (solver.py:237-248)."""
    bysize = {}
    for blk in blocks:
        bysize.setdefault(len(blk.vert_ids), []).append(blk)
    grouped = []
    for s in sorted(bysize):
        fam = bysize[s]
        grouped.append((np.stack([b.hess for b in fam]), np.stack([b.vert_ids for b in fam])))
    return grouped


def _ptr_array(tensors):
    arr = (C.c_void_p * max(len(tensors), 1))()
    for i, t in enumerate(tensors):
        arr[i] = t.data_ptr() if t is not None and t.numel() else None
    return arr


class NewtonSystem:
    """The assembled Newton matrix of one scene on one GPU.

    ``masses`` (N,), ``fixed`` (N,) bool.  Call ``set_pattern`` whenever the contact set
    changes (symbolic phase: sort-by-key, pattern, source runs), then ``assemble`` for every
    new set of block values (numeric phase: deterministic segmented sums, no atomics).
    """

    def __init__(self, masses, fixed):
        self.masses = device.to_device(masses, np.float64)
        self.n = int(self.masses.shape[0])
        fx = np.ascontiguousarray(np.asarray(device.to_host(fixed) if not isinstance(fixed, np.ndarray) else fixed))
        self.fixed = device.to_device(fx.astype(np.uint8))
        if self.fixed.shape[0] != self.n:
            raise ValueError("masses and fixed disagree on the vertex count")
        self._h = C.c_void_p()
        _lib.check(_lib.lib().b200ipc_assembly_create(C.byref(self._h)), "assembly_create")
        self.nnzb = 0
        self.rowptr = self.colidx = self.vals = self.pinv = None
        self._fam = []        # [(s, nb, vids tensor)]
        self._tiled = []      # per family: dense blocks arrive sub-block-major
        self._pcg_ws = None
        self._mas, self._mas_ordered, self._mas_levels, self._mas_stale = None, False, 0, True

    def set_numeric_variant(self, variant):
        """0 = automatic (default: per-block runs when applicable), 1 = per-block runs, 4 = row-wise
        (see include/b200ipc.h)."""
        _lib.check(_lib.lib().b200ipc_assembly_set_variant(self._h, int(variant)), "assembly_set_variant")

    def set_symbolic_mode(self, mode):
        """0 = row-wise symbolic phase (default; sort path when a row has > 256 columns), 1 = sort by key."""
        _lib.check(_lib.lib().b200ipc_assembly_set_symbolic(self._h, int(mode)), "assembly_set_symbolic")

    def stats(self):
        """{'symbolic': 'rows' | 'sort', 'max_row': longest block row (-1 = not measured), 'nnzb', 'sources'}."""
        out = (C.c_int64 * 4)()
        _lib.check(_lib.lib().b200ipc_assembly_stats(self._h, out), "assembly_stats")
        return {"symbolic": {1: "sort", 2: "rows"}.get(int(out[0]), "?"), "max_row": int(out[1]),
                "nnzb": int(out[2]), "sources": int(out[3])}

    def close(self):
        if getattr(self, "_mas", None) is not None and self._mas:
            _lib.lib().b200ipc_mas_destroy(self._mas)
            self._mas = None
        if getattr(self, "_h", None) is not None and self._h:
            _lib.lib().b200ipc_assembly_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- symbolic ---------------------------------------------------------------------------
    def set_pattern(self, families, tiled=None):
        """``families``: iterable of (s, vids) with vids an (nb, s) int64 array/tensor.  ``tiled``: one flag per
        family -- ``assemble`` will be given that family's dense blocks sub-block-major, (nb,s,s,3,3)
        (``stencils.evaluate(..., hess_layout="subblock")``), instead of the reference's (nb,3s,3s)."""
        families = list(families)
        flags = [False] * len(families) if tiled is None else [bool(t) for t in tiled]
        if len(flags) != len(families):
            raise ValueError("one tiled flag per family")
        flags = [t for t, (s, vids) in zip(flags, families) if len(vids)]   # empty families are dropped below
        mask = sum(1 << f for f, t in enumerate(flags) if t)
        _lib.check(_lib.lib().b200ipc_assembly_set_layout(self._h, mask), "assembly_set_layout")
        self._tiled = flags
        fam = []
        for s, vids in families:
            v = device.to_device(vids, np.int64)
            if v.dim() != 2 or v.shape[1] != s or s not in (2, 3, 4):
                raise ValueError("family vids must be (nb, s) with s in {2, 3, 4}")
            if v.shape[0]:
                fam.append((int(s), int(v.shape[0]), v))
        self._fam = fam
        nf = len(fam)
        fs = (C.c_int32 * max(nf, 1))(*[f[0] for f in fam])
        fnb = (C.c_int64 * max(nf, 1))(*[f[1] for f in fam])
        nnzb = C.c_int64(0)
        _lib.check(_lib.lib().b200ipc_assemble_symbolic(self._h, self.n, device.ptr(self.fixed), nf, fs, fnb,
                                                        _ptr_array([f[2] for f in fam]), C.byref(nnzb),
                                                        device.stream()), "assemble_symbolic")
        self.nnzb = int(nnzb.value)
        self.rowptr = device.empty((self.n + 1,), np.int32)
        self.colidx = device.empty((self.nnzb,), np.int32)
        _lib.check(_lib.lib().b200ipc_assembly_pattern(self._h, device.ptr(self.rowptr), device.ptr(self.colidx),
                                                       device.stream()), "assembly_pattern")
        self.vals = device.empty((self.nnzb, 3, 3))
        self.pinv = None
        return self.nnzb

    def _match(self, tensors, width):
        if len(tensors) != len(self._fam):
            raise ValueError("one array per non-empty family, in set_pattern order")
        out = []
        for (s, nb, _), t in zip(self._fam, tensors):
            t = device.to_device(t, np.float64)
            if t.shape[0] != nb or t.numel() != nb * width(s):
                raise ValueError("family array does not match the pattern")
            out.append(t)
        return out

    # -- numeric ----------------------------------------------------------------------------
    def assemble(self, fam_hess):
        """vals = diag(m I) + segmented sums of the families' blocks (fixed rows: identity)."""
        hs = self._match([h for h in fam_hess if h is not None and len(h)], lambda s: 9 * s * s)
        for h, t in zip(hs, self._tiled):
            if (h.dim() == 5) != t:    # same byte count either way: a mix-up would assemble a wrong matrix silently
                raise ValueError("family blocks are %s but the pattern was set for %s" %
                                 (("sub-block-major", "row-major") if h.dim() == 5 else ("row-major", "sub-block-major")))
        _lib.check(_lib.lib().b200ipc_assemble_numeric(self._h, device.ptr(self.masses), _ptr_array(hs),
                                                       device.ptr(self.vals), device.stream()), "assemble_numeric")
        self.pinv = None
        self._mas_stale = True
        return self.vals

    FACTOR_INDEX_BITS = 27   # element index field of the factor descriptors (assembly.cu factor_desc_kernel)

    @classmethod
    def factors_fit(cls, family_counts):
        """True when ``assemble_from_factors`` can address every family: nb * 3 s below 2**27 elements
        (``family_counts``: {s: nb}); beyond that the dense path (``assemble``) applies."""
        return all(int(nb) * 3 * int(s) < (1 << cls.FACTOR_INDEX_BITS) for s, nb in family_counts.items())

    def assemble_from_factors(self, fam_fac):
        """Same matrix from the rank-1 factors z of the barrier blocks (hess = z z^T), without the
        dense blocks: the gathers read 24 s instead of 72 s^2 bytes per block and stay in L2."""
        fs = self._match([z for z in fam_fac if z is not None and len(z)], lambda s: 3 * s)
        _lib.check(_lib.lib().b200ipc_assemble_numeric_factors(self._h, device.ptr(self.masses), _ptr_array(fs),
                                                               device.ptr(self.vals), device.stream()),
                   "assemble_numeric_factors")
        self.pinv = None
        self._mas_stale = True
        return self.vals

    def gradient(self, x, x_tilde, fam_grad):
        """M (x - x~) + scattered block gradients, fixed rows zero (solver.py:218-226)."""
        gs = self._match([g for g in fam_grad if g is not None and len(g)], lambda s: 3 * s)
        dx, dxt = device.to_device(x, np.float64), device.to_device(x_tilde, np.float64)
        out = device.empty((3 * self.n,))
        _lib.check(_lib.lib().b200ipc_scatter_gradient(self._h, device.ptr(self.masses), device.ptr(dx),
                                                       device.ptr(dxt), _ptr_array(gs), device.ptr(out),
                                                       device.stream()), "scatter_gradient")
        return out

    def spmv(self, x, out=None):
        dx = device.to_device(x, np.float64)
        y = device.empty((3 * self.n,)) if out is None else out
        _lib.check(_lib.lib().b200ipc_bsr_spmv(self.n, self.nnzb, device.ptr(self.rowptr), device.ptr(self.colidx),
                                               device.ptr(self.vals), device.ptr(dx), device.ptr(y),
                                               device.stream()), "bsr_spmv")
        return y

    def block_jacobi(self):
        if self.pinv is None:
            self.pinv = device.empty((self.n, 3, 3))
            _lib.check(_lib.lib().b200ipc_block_jacobi(self.n, device.ptr(self.rowptr), device.ptr(self.colidx),
                                                       device.ptr(self.vals), device.ptr(self.pinv),
                                                       device.stream()), "block_jacobi")
        return self.pinv

    # -- multilevel additive Schwarz ------------------------------------------
    def mas_order(self, positions=None):
        """Domain order of the MAS preconditioner: Morton order of ``positions`` (N,3), or index order."""
        if self._mas is None:
            self._mas = C.c_void_p()
            _lib.check(_lib.lib().b200ipc_mas_create(C.byref(self._mas)), "mas_create")
        x = None if positions is None else device.to_device(positions, np.float64)
        _lib.check(_lib.lib().b200ipc_mas_order(self._mas, self.n, device.ptr(x) if x is not None else None,
                                                device.stream()), "mas_order")
        self._mas_ordered, self._mas_levels = True, 0

    def mas_rank(self):
        rank = device.empty((self.n,), np.int32)
        _lib.check(_lib.lib().b200ipc_mas_get_order(self._mas, device.ptr(rank), device.stream()), "mas_get_order")
        return rank

    def mas_setup(self, levels=1):
        """Gather and invert the domain matrices of the current ``vals`` (call after every ``assemble``)."""
        if not self._mas_ordered:
            self.mas_order(None)
        _lib.check(_lib.lib().b200ipc_mas_setup(self._mas, self.n, self.nnzb, device.ptr(self.rowptr),
                                                device.ptr(self.colidx), device.ptr(self.vals), device.ptr(self.fixed),
                                                int(levels), device.stream()), "mas_setup")
        self._mas_levels = int(levels)

    def mas_apply(self, r):
        dr = device.to_device(r, np.float64)
        z = device.empty((3 * self.n,))
        _lib.check(_lib.lib().b200ipc_mas_apply(self._mas, device.ptr(dr), device.ptr(z), device.stream()), "mas_apply")
        return z

    def pcg(self, rhs, rel_tol, max_iters, preconditioner="block_jacobi", mas_levels=1):
        """Returns (d tensor (3N), iters, converged, delta0, delta_new).

        ``preconditioner``: "block_jacobi" (the reference's, solver.py:265-276; default) or "mas" (multilevel
        additive Schwarz over the domains of ``mas_order``; the loop still stops on the reference's
        block-Jacobi-norm rule, and delta0 / delta_new are reported in that norm)."""
        pinv = self.block_jacobi()
        drhs = device.to_device(rhs, np.float64)
        d = device.empty((3 * self.n,))
        if preconditioner == "mas":
            if self._mas_levels != int(mas_levels) or self._mas_stale:
                self.mas_setup(mas_levels)
                self._mas_stale = False
            nbytes = int(_lib.lib().b200ipc_pcg_mas_workspace_bytes(self.n))
            if self._pcg_ws is None or self._pcg_ws.numel() * 8 < nbytes:
                self._pcg_ws = device.empty(((nbytes + 7) // 8,))
            res = _lib.PcgResult()
            _lib.check(_lib.lib().b200ipc_pcg_mas(self._mas, self.n, self.nnzb, device.ptr(self.rowptr),
                                                  device.ptr(self.colidx), device.ptr(self.vals), device.ptr(pinv),
                                                  device.ptr(self.fixed), device.ptr(drhs), device.ptr(d), float(rel_tol),
                                                  int(max_iters), device.ptr(self._pcg_ws), nbytes, C.byref(res),
                                                  device.stream()), "pcg_mas")
            return d, int(res.iters), bool(res.converged), float(res.delta0), float(res.delta_new)
        if preconditioner != "block_jacobi":
            raise ValueError("preconditioner must be 'block_jacobi' or 'mas'")
        nbytes = int(_lib.lib().b200ipc_pcg_workspace_bytes(self.n))
        if self._pcg_ws is None or self._pcg_ws.numel() * 8 < nbytes:
            self._pcg_ws = device.empty(((nbytes + 7) // 8,))
        res = _lib.PcgResult()
        _lib.check(_lib.lib().b200ipc_pcg(self.n, self.nnzb, device.ptr(self.rowptr), device.ptr(self.colidx),
                                          device.ptr(self.vals), device.ptr(pinv), device.ptr(self.fixed),
                                          device.ptr(drhs), device.ptr(d), float(rel_tol), int(max_iters),
                                          device.ptr(self._pcg_ws), nbytes, C.byref(res), device.stream()), "pcg")
        return d, int(res.iters), bool(res.converged), float(res.delta0), float(res.delta_new)

    def to_scipy_like(self):
        """(rowptr, colidx, vals) as host arrays."""
        return device.to_host(self.rowptr), device.to_host(self.colidx), device.to_host(self.vals)


def _system_from_grouped(grouped, masses, fixed, variant=0):
    sysm = NewtonSystem(masses, fixed)
    sysm.set_numeric_variant(variant)
    fams = [(int(v.shape[1]), v) for _, v in grouped if len(v)]
    sysm.set_pattern(fams)
    sysm.assemble([h for h, v in grouped if len(v)])
    return sysm


def assemble_bsr(grouped, masses, fixed):
    """Assembled matrix of ``grouped`` blocks as host BSR arrays (rowptr, colidx, vals)."""
    sysm = _system_from_grouped(grouped, masses, fixed)
    try:
        return sysm.to_scipy_like()
    finally:
        sysm.close()


def matvec_matrix_free(grouped, masses, fixed, v):
    """A @ v without assembling A (solver.py:251-262); host arrays in and out."""
    masses = np.asarray(masses, dtype=np.float64)
    n = masses.shape[0]
    d_m = device.to_device(masses)
    d_f = device.to_device(np.asarray(fixed).astype(np.uint8))
    d_v = device.to_device(np.asarray(v, dtype=np.float64))
    vin, out = device.empty((3 * n,)), device.empty((3 * n,))
    L = _lib.lib()
    _lib.check(L.b200ipc_matvec_begin(n, device.ptr(d_m), device.ptr(d_f), device.ptr(d_v), device.ptr(vin),
                                      device.ptr(out), device.stream()), "matvec_begin")
    keep = []
    for hess, vids in grouped:
        if len(vids) == 0:
            continue
        d_h, d_i = device.to_device(hess, np.float64), device.to_device(vids, np.int64)
        keep.append((d_h, d_i))
        matvec_blocks_device(d_h, d_i, vin, out)
    _lib.check(L.b200ipc_matvec_end(n, device.ptr(d_f), device.ptr(d_v), device.ptr(out), device.stream()),
               "matvec_end")
    return device.to_host(out)


def block_jacobi_preconditioner(grouped, masses, fixed):
    """Inverted per-vertex 3x3 diagonal blocks of the assembled system (solver.py:265-276)."""
    sysm = _system_from_grouped(grouped, masses, fixed)
    try:
        return device.to_host(sysm.block_jacobi())
    finally:
        sysm.close()


def pcg_solve(grouped, masses, fixed, rhs, rel_tol, max_iters):
    """Block-Jacobi PCG (solver.py:279-315): returns (d, iters, converged)."""
    sysm = _system_from_grouped(grouped, masses, fixed)
    try:
        d, iters, ok, _, _ = sysm.pcg(np.asarray(rhs, dtype=np.float64), rel_tol, max_iters)
        return device.to_host(d), iters, ok
    finally:
        sysm.close()


_STEPPER_NAMES = ("SolverConfig", "StepStats", "SimState", "newton_step", "advance_time_step", "MODE_GIPC",
                  "MODE_REFERENCE")


def __getattr__(name):
    """The reference keeps the time stepper in the same module (solver.py:32-235, :316-422); here it
    lives in ``stepper`` and is reachable under the reference's import path as well."""
    if name in _STEPPER_NAMES:
        from . import stepper

        return getattr(stepper, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
