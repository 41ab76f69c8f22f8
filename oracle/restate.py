"""CPU restatement of the reference smoother for line and plane blocks.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1208_1975_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` leg use it, and only as the checker.

It restates, in vectorised numpy, the algorithm of the reference package
``patchsmooth`` 0.1.0 (``/root/reference/pkg/src/patchsmooth``) for the hot
path: block Jacobi and serial (lexicographic) block Gauss-Seidel with exact
x-line blocks ``(>=nx, 1, 1)`` and exact xy-plane blocks ``(>=nx, >=ny, 1)``
of the constant-coefficient 7-point stencil, on single patches and on
multi-patch levels.  The citations below name the reference lines each
function follows.

The only deliberate departure from the reference is how the exact block
inverse is applied.  The reference multiplies by a dense LU-built inverse
(``blocklinalg.py:50-105``); here the same exact inverse is applied as a
Thomas solve (lines) or a DST-I diagonalisation in x followed by Thomas solves
in y (planes).  Both are exact; they differ from the dense matvec only by
rounding (<=5e-16 relative, pinned against the reference itself by
``tests/test_oracle_golden.py`` through the fixtures in ``tests/golden/``,
which ``oracle/make_golden.py`` generates by running the reference).
"""

from __future__ import annotations

import itertools
import math

import numpy as np

# stencil.py:42-49 -- neighbour offsets in the fixed face order.
FACE_OFFSETS = ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1))

DEFAULT_CENTER = 6.0
DEFAULT_FACES = (-1.0, -1.0, -1.0, -1.0, -1.0, -1.0)


# --------------------------------------------------------------------------
# data: a patch is (dims, origin, two padded F-order buffers, interior f)
# --------------------------------------------------------------------------
class OPatch:
    """grid.py:153-217 restated: padded u/v buffers with a role flag, plus f."""

    def __init__(self, dims, origin=(0, 0, 0)):
        self.dims = tuple(int(n) for n in dims)
        self.origin = tuple(int(o) for o in origin)
        pad = tuple(n + 2 for n in self.dims)
        self.bufs = [np.zeros(pad, order="F"), np.zeros(pad, order="F")]
        self.active = 0
        self.f = np.zeros(self.dims, order="F")

    @property
    def u(self):
        return self.bufs[self.active]

    @property
    def other(self):
        return self.bufs[1 - self.active]

    @property
    def interior(self):
        return self.u[1:-1, 1:-1, 1:-1]

    def swap(self):  # grid.py:204-206
        self.active = 1 - self.active

    @property
    def global_box(self):
        return tuple((o, o + n) for o, n in zip(self.origin, self.dims))


def find_abutments(patches):
    """grid.py:429-465 restated: symmetric face-abutment copies.

    Returns a list of (src, dst, src_lo, dst_lo, extent) tuples in the
    reference's order (pairs in combinations order, forward then mirror).
    """
    copies = []
    for ia, ib in itertools.combinations(range(len(patches)), 2):
        a, b = patches[ia], patches[ib]
        boxes = list(zip(a.global_box, b.global_box))
        overlaps = []
        for (alo, ahi), (blo, bhi) in boxes:
            lo, hi = max(alo, blo), min(ahi, bhi)
            overlaps.append((lo, hi) if lo < hi else None)
        if all(o is not None for o in overlaps):
            raise ValueError(f"patches {ia} and {ib} overlap")
        for axis in range(3):
            (a_lo, a_hi), (b_lo, b_hi) = boxes[axis]
            trans = [overlaps[ax] for ax in range(3) if ax != axis]
            if any(t is None for t in trans):
                continue
            if a_hi == b_lo:
                low, high, ilow, ihigh = a, b, ia, ib
            elif b_hi == a_lo:
                low, high, ilow, ihigh = b, a, ib, ia
            else:
                continue
            src_lo, dst_lo, ext = [0] * 3, [0] * 3, [0] * 3
            src_lo[axis] = low.dims[axis] - 1
            dst_lo[axis] = -1
            ext[axis] = 1
            t = iter(trans)
            for ax in range(3):
                if ax == axis:
                    continue
                t_lo, t_hi = next(t)
                src_lo[ax] = t_lo - low.origin[ax]
                dst_lo[ax] = t_lo - high.origin[ax]
                ext[ax] = t_hi - t_lo
            fwd = (ilow, ihigh, tuple(src_lo), tuple(dst_lo), tuple(ext))
            # grid.py:_mirror (:355-381): high's low layer feeds low's high ghost
            m_src_lo, m_dst_lo = list(dst_lo), list(src_lo)
            m_src_lo[axis] = 0
            m_dst_lo[axis] = low.dims[axis]
            mir = (ihigh, ilow, tuple(m_src_lo), tuple(m_dst_lo), tuple(ext))
            copies.append(fwd)
            copies.append(mir)
    return copies


class OLevel:
    """grid.py:468-520 restated: patches plus derived adjacency."""

    def __init__(self, patches, adjacency=None):
        self.patches = list(patches)
        self.adjacency = find_abutments(self.patches) if adjacency is None else list(adjacency)

    def refresh_ghosts(self):  # grid.py:507-517
        for p in self.patches:
            fill_physical_ghosts(p.u)
        exchange_interface_ghosts(self)


def fill_physical_ghosts(u):
    """grid.py:311-330: ghost = -adjacent interior, axis by axis x, y, z."""
    u[0, :, :] = -u[1, :, :]
    u[-1, :, :] = -u[-2, :, :]
    u[:, 0, :] = -u[:, 1, :]
    u[:, -1, :] = -u[:, -2, :]
    u[:, :, 0] = -u[:, :, 1]
    u[:, :, -1] = -u[:, :, -2]
    return u


def exchange_interface_ghosts(level):
    """grid.py:523-547: snapshot all sources, then write all ghosts."""
    staged = []
    for src, dst, src_lo, dst_lo, ext in level.adjacency:
        sl = tuple(slice(l + 1, l + e + 1) for l, e in zip(src_lo, ext))
        staged.append((dst, dst_lo, ext, level.patches[src].u[sl].copy()))
    for dst, dst_lo, ext, data in staged:
        sl = tuple(slice(l + 1, l + e + 1) for l, e in zip(dst_lo, ext))
        level.patches[dst].u[sl] = data
    return level


# --------------------------------------------------------------------------
# residual (stencil.py:93-112) -- same operation order, so bitwise equal
# --------------------------------------------------------------------------
def residual(u, f, center=DEFAULT_CENTER, faces=DEFAULT_FACES, lo=(0, 0, 0), ext=None):
    """f - A u on the interior box [lo, lo+ext), F-order like u.

    acc = center*u, then acc += face_d * u[shift_d] in the order
    -x,+x,-y,+y,-z,+z, then r = f - acc (stencil.py:106-111).
    """
    if ext is None:
        ext = f.shape
    c = tuple(slice(l + 1, l + e + 1) for l, e in zip(lo, ext))
    acc = center * u[c]
    for coef, off in zip(faces, FACE_OFFSETS):
        sh = tuple(slice(s.start + d, s.stop + d) for s, d in zip(c, off))
        acc += coef * u[sh]
    fs = tuple(slice(l, l + e) for l, e in zip(lo, ext))
    return f[fs] - acc


def residual_norm(level, center=DEFAULT_CENTER, faces=DEFAULT_FACES, exact=True):
    """smoother.py:96-109: sqrt of the exactly rounded sum of r^2."""
    if exact:
        terms = []
        for p in level.patches:
            r = residual(p.u, p.f, center, faces)
            terms.extend(np.square(r).ravel().tolist())
        return math.sqrt(math.fsum(terms))
    s = 0.0
    for p in level.patches:
        r = residual(p.u, p.f, center, faces)
        s += float(np.sum(np.square(r), dtype=np.float64))
    return math.sqrt(s)


# --------------------------------------------------------------------------
# exact block solves
# --------------------------------------------------------------------------
def thomas_factors(n, diag, lower, upper):
    """LU factors of tridiag(lower, diag, upper) of order n (no pivoting).

    Returns (cp, inv_m): cp[i] = upper * inv_m[i], inv_m[i] = 1/(diag - lower*cp[i-1]).
    """
    cp = np.empty(n)
    inv_m = np.empty(n)
    prev = 0.0
    for i in range(n):
        m = diag - lower * prev
        inv_m[i] = 1.0 / m
        cp[i] = upper * inv_m[i]
        prev = cp[i]
    return cp, inv_m


def thomas_solve(r, axis, diag, lower, upper):
    """Solve tridiag(lower, diag, upper) x = r along ``axis`` for every line.

    ``diag`` may be a scalar or an array broadcastable against the lines
    (one diagonal per line, used by the plane solve's modal systems).
    """
    r = np.moveaxis(np.asarray(r, dtype=np.float64), axis, 0)
    n = r.shape[0]
    diag = np.asarray(diag, dtype=np.float64)
    x = np.empty_like(r)
    cp = np.empty((n,) + np.broadcast_shapes(diag.shape, r.shape[1:]))
    prev_c = np.zeros_like(cp[0])
    prev_d = np.zeros(r.shape[1:])
    for i in range(n):
        inv = 1.0 / (diag - lower * prev_c)
        cp[i] = upper * inv
        x[i] = (r[i] - lower * prev_d) * inv
        prev_c, prev_d = cp[i], x[i]
    for i in range(n - 2, -1, -1):
        x[i] = x[i] - cp[i] * x[i + 1]
    return np.moveaxis(x, 0, axis)


def line_solve(r, center=DEFAULT_CENTER, faces=DEFAULT_FACES):
    """Exact inverse of the closure-free line block (stencil.py:115-138 with
    extent (nx,1,1)): tridiag(faces[0], center, faces[1]) along x."""
    return thomas_solve(r, 0, center, faces[0], faces[1])


def dst_basis(n):
    """Orthonormal DST-I basis Q[p, i] = sqrt(2/(n+1)) sin(pi (p+1)(i+1)/(n+1))
    and eigen-offsets cos(pi (i+1)/(n+1)); Q is symmetric and Q @ Q = I."""
    idx = np.arange(1, n + 1)
    q = np.sqrt(2.0 / (n + 1)) * np.sin(np.pi * np.outer(idx, idx) / (n + 1))
    cosv = np.cos(np.pi * idx / (n + 1))
    return q, cosv


def plane_solve(r, center=DEFAULT_CENTER, faces=DEFAULT_FACES):
    """Exact inverse of the closure-free plane block (stencil.py:115-138 with
    extent (nx,ny,1)).  Requires faces[0] == faces[1] (symmetric x coupling):
    x is diagonalised by DST-I, leaving one tridiagonal system in y per x-mode
    with diagonal center + 2*faces[0]*cos(pi i/(nx+1))."""
    if faces[0] != faces[1]:
        raise ValueError("plane solve needs symmetric x faces")
    nx = r.shape[0]
    q, cosv = dst_basis(nx)
    rh = np.tensordot(q, r, axes=([1], [0]))  # modes along axis 0
    # thomas along y (axis 1); the remaining line axes are (x-mode, z...)
    diag = (center + 2.0 * faces[0] * cosv).reshape((nx,) + (1,) * (r.ndim - 2))
    xh = thomas_solve(rh, 1, diag, faces[2], faces[3])
    return np.tensordot(q, xh, axes=([1], [0]))


def _is_line(dims, block):
    return block[0] >= dims[0] and block[1] == 1 and block[2] == 1


def _is_plane(dims, block):
    return block[0] >= dims[0] and block[1] >= dims[1] and block[2] == 1


def block_kind(dims, block):
    """Classify block_dims (grid.py:298-306 truncation): one block per line,
    per plane, or general boxes (the paper's cubic blocks)."""
    if _is_line(dims, block):
        return "line"
    if _is_plane(dims, block):
        return "plane"
    return "box"


def box_matrix(ext, center=DEFAULT_CENTER, faces=DEFAULT_FACES):
    """assemble_block_matrix (stencil.py:115-138): the closure-free operator of
    one block, cells x fastest; couplings leaving the block are dropped."""
    ex, ey, ez = ext
    n = ex * ey * ez
    a = np.zeros((n, n))
    for k in range(ez):
        for j in range(ey):
            for i in range(ex):
                row = i + ex * (j + ey * k)
                a[row, row] = center
                for coef, (dx, dy, dz) in zip(faces, FACE_OFFSETS):
                    ii, jj, kk = i + dx, j + dy, k + dz
                    if 0 <= ii < ex and 0 <= jj < ey and 0 <= kk < ez:
                        a[row, ii + ex * (jj + ey * kk)] = coef
    return a


_BOX_INV = {}


def box_inverse(ext, center=DEFAULT_CENTER, faces=DEFAULT_FACES):
    """Dense exact inverse per block shape (invert_dense, blocklinalg.py:50-87)."""
    key = (tuple(ext), float(center), tuple(float(f) for f in faces))
    inv = _BOX_INV.get(key)
    if inv is None:
        inv = np.linalg.inv(box_matrix(ext, center, faces))
        _BOX_INV[key] = inv
    return inv


def box_ranges(dims, block):
    """decompose_blocks (grid.py:286-308): lexicographic, x fastest."""
    counts = [-(-n // b) for n, b in zip(dims, block)]
    for kz in range(counts[2]):
        for ky in range(counts[1]):
            for kx in range(counts[0]):
                lo = (kx * block[0], ky * block[1], kz * block[2])
                yield lo, tuple(min(b, n - l) for b, n, l in zip(block, dims, lo))


def box_update(p, lo, ext, omega, center, faces, dst):
    """block_update (smoother.py:90-93) of one box: dst_b = u_b + omega Ainv r_b
    with r_b = block_residual of the current u (cells x fastest)."""
    r = residual(p.u, p.f, center, faces, lo=lo, ext=ext)
    x = box_inverse(ext, center, faces) @ r.transpose(2, 1, 0).ravel()
    sl = tuple(slice(l + 1, l + e + 1) for l, e in zip(lo, ext))
    dst[sl] = p.u[sl] + omega * x.reshape(ext[2], ext[1], ext[0]).transpose(2, 1, 0)


# --------------------------------------------------------------------------
# sweeps
# --------------------------------------------------------------------------
def jacobi_step(level, block, omega, center=DEFAULT_CENTER, faces=DEFAULT_FACES):
    """smoother.py:138-153: v = u + omega * Ainv r from one snapshot of u,
    then swap buffers and refresh ghosts."""
    for p in level.patches:
        kind = block_kind(p.dims, block)
        if kind == "box":
            for lo, ext in box_ranges(p.dims, block):
                box_update(p, lo, ext, omega, center, faces, p.other)
            continue
        r = residual(p.u, p.f, center, faces)
        x = line_solve(r, center, faces) if kind == "line" else plane_solve(r, center, faces)
        p.other[1:-1, 1:-1, 1:-1] = p.interior + omega * x
    for p in level.patches:
        p.swap()
    level.refresh_ghosts()


def gs_step(level, block, omega, center=DEFAULT_CENTER, faces=DEFAULT_FACES):
    """smoother.py:156-169 under the serial strategy (runtime.py:164-168):
    lexicographic in-place block updates, patches in order, ghosts lagged to
    step end.  Lines (j,k) run as wavefronts d = j+k -- every line of one
    wavefront reads only lines of earlier wavefronts or not-yet-updated ones,
    exactly as in the lexicographic order, so this is the same arithmetic."""
    for p in level.patches:
        kind = block_kind(p.dims, block)
        nx, ny, nz = p.dims
        u = p.u
        if kind == "box":  # lexicographic blocks, in place
            for lo, ext in box_ranges(p.dims, block):
                box_update(p, lo, ext, omega, center, faces, u)
            continue
        if kind == "plane":
            for k in range(nz):
                r = residual(u, p.f, center, faces, lo=(0, 0, k), ext=(nx, ny, 1))
                x = plane_solve(r, center, faces)
                u[1:-1, 1:-1, k + 1 : k + 2] = u[1:-1, 1:-1, k + 1 : k + 2] + omega * x
            continue
        for d in range(ny + nz - 1):
            js = np.arange(max(0, d - nz + 1), min(ny, d + 1))
            ks = d - js
            jj, kk = js + 1, ks + 1
            acc = center * u[1:-1, jj, kk]
            acc += faces[0] * u[0:-2, jj, kk]
            acc += faces[1] * u[2:, jj, kk]
            acc += faces[2] * u[1:-1, jj - 1, kk]
            acc += faces[3] * u[1:-1, jj + 1, kk]
            acc += faces[4] * u[1:-1, jj, kk - 1]
            acc += faces[5] * u[1:-1, jj, kk + 1]
            r = p.f[:, js, ks] - acc
            x = line_solve(r, center, faces)
            u[1:-1, jj, kk] = u[1:-1, jj, kk] + omega * x
    level.refresh_ghosts()


def smooth(level, scheme, block, omega=None, steps=1, center=DEFAULT_CENTER,
           faces=DEFAULT_FACES, exact_norm=True):
    """smoother.py:197-214: refresh, history[0], then steps x (step, norm)."""
    if omega is None:
        omega = 0.8 if scheme == "block_jacobi" else 1.0  # smoother.py:51
    step = jacobi_step if scheme == "block_jacobi" else gs_step
    level.refresh_ghosts()
    hist = [residual_norm(level, center, faces, exact_norm)]
    for _ in range(steps):
        step(level, block, omega, center, faces)
        hist.append(residual_norm(level, center, faces, exact_norm))
    return hist


def seed_initial_guess(level, seed):
    """bench.py:141-146: interior ~ U[0,1) from one generator, patch order."""
    rng = np.random.default_rng(seed)
    for p in level.patches:
        p.interior[...] = rng.random(p.dims)
    return level


def lattice_level(counts, size):
    """A counts[0] x counts[1] x counts[2] lattice of equal patches (the AMR
    config C4 is counts=(4,4,4), size=(128,128,128)); patch order x fastest."""
    patches = []
    for c in range(counts[2]):
        for b in range(counts[1]):
            for a in range(counts[0]):
                patches.append(OPatch(size, (a * size[0], b * size[1], c * size[2])))
    return OLevel(patches)
