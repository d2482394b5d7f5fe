"""Host-side mirror of the reference's stencil types plus the SoA stencil table.

``StencilKind`` / ``ContactStencil`` / ``DistanceResult`` keep the reference's names and
fields (``/root/reference/pkg/src/tetipc/proximity.py:27-96``) so host code written against
``tetipc`` reads the same.  The GPU path works on ``StencilTable``: one row per contact in
the reference's list order, stored as flat arrays.
"""

import enum
from dataclasses import dataclass

import numpy as np


class ProximityError(ValueError):
    pass


class StencilKind(enum.Enum):
    POINT_POINT = "point-point"
    POINT_EDGE = "point-edge"
    POINT_TRIANGLE = "point-triangle"
    EDGE_EDGE = "edge-edge"
    EDGE_EDGE_PARALLEL = "edge-edge-parallel"
    POINT_EDGE_PARALLEL = "point-edge-parallel"
    POINT_POINT_PARALLEL = "point-point-parallel"


PARALLEL_KINDS = frozenset(
    {StencilKind.EDGE_EDGE_PARALLEL, StencilKind.POINT_EDGE_PARALLEL, StencilKind.POINT_POINT_PARALLEL}
)

#: kind code = rank of the enum value string = position in the reference's sorted contact list
KIND_ORDER = tuple(sorted(StencilKind, key=lambda k: k.value))
KIND_CODE = {k: i for i, k in enumerate(KIND_ORDER)}
EE, EEP, PE, PEP, PP, PPP, PT = range(7)
KIND_SIZE = np.array([4, 4, 3, 4, 2, 4, 4], dtype=np.int64)
IS_PARALLEL = np.array([False, True, False, True, False, True, False])
#: order of kinds inside the 12x12 family of group_blocks (list order restricted to s = 4)
FAMILY4_KINDS = (EE, EEP, PEP, PPP, PT)

SIMPLEX_DIM = {
    StencilKind.POINT_POINT: 1,
    StencilKind.POINT_EDGE: 2,
    StencilKind.POINT_TRIANGLE: 3,
    StencilKind.EDGE_EDGE: 3,
    StencilKind.EDGE_EDGE_PARALLEL: 3,
    StencilKind.POINT_EDGE_PARALLEL: 3,
    StencilKind.POINT_POINT_PARALLEL: 3,
}


@dataclass(frozen=True)
class ContactStencil:
    """Typed contact pair, field-compatible with the reference (proximity.py:53-83)."""

    kind: StencilKind
    verts: tuple
    eps_x: float = None
    edge_pair: tuple = None
    sub: tuple = None
    origin: tuple = None

    def __post_init__(self):
        expected = int(KIND_SIZE[KIND_CODE[self.kind]])
        if len(self.verts) != expected:
            raise ProximityError(f"{self.kind} expects {expected} vertices, got {len(self.verts)}")
        if self.kind in PARALLEL_KINDS and not (self.eps_x and self.eps_x > 0.0):
            raise ProximityError("parallel stencils need eps_x > 0")

    def sort_key(self):
        return (self.kind.value, self.verts, self.origin or ())


@dataclass
class DistanceResult:
    d2: float
    grad_d2: np.ndarray
    witness: np.ndarray


def pack_sub(local):
    out = 0
    for k, loc in enumerate(local):
        out |= (int(loc) & 3) << (2 * k)
    return out


_SUB_LEN = (0, 4, 0, 3, 0, 2, 0)
_ORIGIN_TAG = {"ee": 1, "vt": 2}
_ORIGIN_NAME = {1: "ee", 2: "vt"}


@dataclass
class StencilTable:
    """Kind-sorted SoA contact list.

    kind (n,) u8, verts (n,4) i32 (-1 padded), sub (n,) u8 (two bits per local index),
    eps_x (n,) f64, origin_type (n,) u8 (0 none, 1 "ee", 2 "vt"), origin (n,4) i32.
    Rows must be sorted by kind; within a kind the reference order is (verts, origin).
    """

    kind: np.ndarray
    verts: np.ndarray
    sub: np.ndarray
    eps_x: np.ndarray
    origin_type: np.ndarray = None
    origin: np.ndarray = None

    def __post_init__(self):
        self.kind = np.ascontiguousarray(self.kind, dtype=np.uint8)
        n = self.kind.shape[0]
        self.verts = np.ascontiguousarray(self.verts, dtype=np.int32).reshape(n, 4)
        self.sub = np.ascontiguousarray(self.sub, dtype=np.uint8).reshape(n)
        self.eps_x = np.ascontiguousarray(self.eps_x, dtype=np.float64).reshape(n)
        if self.origin_type is None:
            self.origin_type = np.zeros(n, np.uint8)
            self.origin = np.full((n, 4), -1, np.int32)
        if n and np.any(np.diff(self.kind.astype(np.int16)) < 0):
            raise ProximityError("stencil table must be sorted by kind")
        if n and int(self.kind.max()) > 6:
            raise ProximityError("bad kind code")

    def __len__(self):
        return int(self.kind.shape[0])

    def kind_offsets(self):
        """(8,) int64 row offsets: rows of kind k are [off[k], off[k+1])."""
        return np.searchsorted(self.kind, np.arange(8), side="left").astype(np.int64)

    def family_rows(self, s):
        """Table rows of the size-``s`` family in ``group_blocks`` order."""
        off = self.kind_offsets()
        kinds = {2: (PP,), 3: (PE,), 4: FAMILY4_KINDS}[s]
        return np.concatenate([np.arange(off[k], off[k + 1]) for k in kinds]) if len(self) else np.zeros(0, np.int64)

    @classmethod
    def from_stencils(cls, stencils, sort=False):
        """Build from ``ContactStencil``-like objects (this package's or the reference's)."""
        stencils = list(stencils)
        if sort:
            stencils.sort(key=lambda s: s.sort_key())
        n = len(stencils)
        kind = np.zeros(n, np.uint8)
        verts = np.full((n, 4), -1, np.int32)
        sub = np.zeros(n, np.uint8)
        eps = np.zeros(n)
        otype = np.zeros(n, np.uint8)
        origin = np.full((n, 4), -1, np.int32)
        for i, st in enumerate(stencils):
            code = KIND_CODE[StencilKind(st.kind.value)]
            kind[i] = code
            verts[i, : len(st.verts)] = st.verts
            if IS_PARALLEL[code]:
                if st.sub is None or len(st.sub) != _SUB_LEN[code]:
                    raise ProximityError("parallel stencil without a matching sub selection")
                sub[i] = pack_sub(st.sub)
                eps[i] = st.eps_x
            if st.origin is not None:
                otype[i] = _ORIGIN_TAG[st.origin[0]]
                origin[i] = st.origin[1:]
        return cls(kind, verts, sub, eps, otype, origin)

    def to_stencils(self):
        out = []
        for i in range(len(self)):
            code = int(self.kind[i])
            kind = KIND_ORDER[code]
            s = int(KIND_SIZE[code])
            verts = tuple(int(v) for v in self.verts[i, :s])
            origin = None
            if self.origin_type[i]:
                origin = (_ORIGIN_NAME[int(self.origin_type[i])],) + tuple(int(v) for v in self.origin[i])
            if IS_PARALLEL[code]:
                sub = tuple((int(self.sub[i]) >> (2 * k)) & 3 for k in range(_SUB_LEN[code]))
                out.append(ContactStencil(kind=kind, verts=verts, eps_x=float(self.eps_x[i]),
                                          edge_pair=(verts[:2], verts[2:]), sub=sub, origin=origin))
            else:
                out.append(ContactStencil(kind=kind, verts=verts, origin=origin))
        return out
