"""CPU oracle for the DistD2 hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / `--impl reference`
legs may import it. The shipped path (`paper_2411_13532_b200`) never imports
anything under `oracle/` and fails loudly when its CUDA library is missing.

It restates, in plain NumPy, the reference package `tds`
(`/root/reference/pkg/src/tds`, pure Python/NumPy) for the functions on the
DistD2 path, keeping the reference's floating-point association order so the
results are bit-identical to the reference (NumPy ufuncs round every
product/sum; no FMA). Parity is PINNED: `tests/test_oracle_golden.py` checks
every function here bit-for-bit against fixtures produced by importing the
reference itself (`tests/golden/make_golden.py`, committed with its output).
One exception, marked where it lives: the open d2/dx2 closures
(`assemble_open_d2`, shifted stencil windows) restate a B200-side EXTENSION
the reference does not have (it raises, compact.py:79-81) -- PARITY UNPINNED,
validated by order of accuracy instead (tests/test_open_d2.py).

Reference anchors (file:line under /root/reference/pkg/src/tds):
  system.py:148-155  SubdomainPartition.balanced     -> balanced_sizes
  system.py:57-71    effective_lower/upper           -> effective_bands
  system.py:158-167  dominance margin                 -> dominance_margin
  compact.py:37-96   weights / assemble               -> interior_weights, assemble
  distributed.py:119-133 local_slice                  -> local_slice
  distributed.py:144-199 preprocess (Alg. 5)          -> preprocess
  distributed.py:205-239 stencil rows / build_rhs     -> build_rhs
  distributed.py:257-276 decouple_fused (Alg. 6)      -> decouple_fused
  distributed.py:279-293 solve_boundary_pair          -> solve_boundary_pair
  distributed.py:296-305 substitute (Alg. 7)          -> substitute
  distributed.py:327-366 distd2_solve                 -> _rank_solve
  distributed.py:380-396 _serial_reference_solve      -> _serial_solve
  distributed.py:399-449 run_distd2                   -> run_distd2
  serial.py:26-56    thomas_solve                     -> thomas_solve
  serial.py:59-90    periodic_thomas_solve            -> periodic_thomas_solve
  layout.py:82-141   transverse order / pack / unpack -> pack, unpack
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np

PIVOT_FLOOR = 1e-300          # serial.py:21
PAIR_DET_FLOOR = 1e-12        # serial.py:22
HALO = 2                      # distributed.py:40


class OracleError(Exception):
    """Raised where the reference raises SingularPivot/SingularPair/..."""


# ---------------------------------------------------------------- system.py

def balanced_sizes(n, p):
    """system.py:148-155 -- first n mod p blocks get one extra row."""
    if p < 1:
        raise ValueError("rank_count must be positive")
    q, extra = divmod(n, p)
    sizes = tuple(q + (1 if k < extra else 0) for k in range(p))
    if any(s < 4 for s in sizes):
        raise ValueError("every subdomain needs at least 4 rows")
    return sizes


def offsets_of(sizes):
    """system.py:141-146."""
    return tuple(int(v) for v in np.concatenate([[0], np.cumsum(sizes)[:-1]]))


def effective_bands(lower, upper, periodic):
    """system.py:57-71 -- open systems ignore the two corner couplings."""
    a = np.array(lower, dtype=np.float64)
    c = np.array(upper, dtype=np.float64)
    if not periodic:
        a[0] = 0.0
        c[-1] = 0.0
    return a, c


def dominance_margin(lower, diag, upper, periodic):
    """system.py:163-167."""
    a, c = effective_bands(lower, upper, periodic)
    return float(np.min(np.abs(diag) - np.abs(a) - np.abs(c)))


# --------------------------------------------------------------- compact.py

def interior_weights(order, a_w, b_w, h):
    """compact.py:37-46 -- width-5 RHS weights at offsets -2..+2."""
    if order == 1:
        return np.array([-b_w / (4 * h), -a_w / (2 * h), 0.0,
                         a_w / (2 * h), b_w / (4 * h)])
    h2 = h * h
    return np.array([b_w / (4 * h2), a_w / h2, -2 * a_w / h2 - b_w / (2 * h2),
                     a_w / h2, b_w / (4 * h2)])


SCHEMES = {
    # compact.py:49-56: (derivative order, alpha, a, b)
    "d1": (1, 1.0 / 3.0, 14.0 / 9.0, 1.0 / 9.0),
    "d2": (2, 2.0 / 11.0, 12.0 / 11.0, 3.0 / 11.0),
}


def assemble(kind, n, h, periodic=True):
    """compact.py:70-96 -> (lower, diag, upper, stencil(n,5))."""
    order, alpha, a_w, b_w = SCHEMES[kind]
    lower = np.full(n, alpha)
    diag = np.ones(n)
    upper = np.full(n, alpha)
    st = np.tile(interior_weights(order, a_w, b_w, h), (n, 1))
    if not periodic:
        if order != 1:
            raise NotImplementedError("open closures exist for d/dx only")
        e0 = np.array([0.0, 0.0, -2.5, 2.0, 0.5])      # compact.py:64-67
        e1 = np.array([0.0, -0.75, 0.0, 0.75, 0.0])
        lower[0], upper[0], st[0] = 0.0, 2.0, e0 / h
        lower[1] = upper[1] = 0.25
        st[1] = e1 / h
        lower[n - 2] = upper[n - 2] = 0.25
        st[n - 2] = e1 / h
        lower[n - 1], upper[n - 1] = 2.0, 0.0
        st[n - 1] = -e0[::-1] / h
    return lower, diag, upper, st


# Open d2/dx2 closures -- a B200-side EXTENSION: the reference raises
# NotImplementedError for non-periodic second derivatives (compact.py:79-81),
# so these rows are PARITY UNPINNED against the reference; they are validated
# by their order of accuracy (tests/test_open_d2.py). Row 0: explicit
# one-sided 5-point formula (offsets 0..4, third-order truncation, no LHS
# coupling); row 1: the fourth-order Pade scheme beta = 1/10 with
# 6/5 (u0 - 2 u1 + u2) / h^2; mirrored at the end. Row 0 / n-1 reach past
# the width-5 window: their stencil window is shifted by +2 / -2.
D2_EDGE0_W = np.array([35.0 / 12.0, -26.0 / 3.0, 19.0 / 2.0, -14.0 / 3.0, 11.0 / 12.0])
D2_EDGE1_BETA = 0.1
D2_EDGE1_W = np.array([0.0, 1.2, -2.4, 1.2, 0.0])


def assemble_open_d2(n, h):
    """-> (lower, diag, upper, stencil(n,5), shift(n,)) of the open d2/dx2."""
    order, alpha, a_w, b_w = SCHEMES["d2"]
    lower = np.full(n, alpha)
    diag = np.ones(n)
    upper = np.full(n, alpha)
    st = np.tile(interior_weights(order, a_w, b_w, h), (n, 1))
    shift = np.zeros(n, dtype=np.int32)
    h2 = h * h
    lower[0], upper[0], st[0], shift[0] = 0.0, 0.0, D2_EDGE0_W / h2, 2
    lower[1] = upper[1] = D2_EDGE1_BETA
    st[1] = D2_EDGE1_W / h2
    lower[n - 2] = upper[n - 2] = D2_EDGE1_BETA
    st[n - 2] = D2_EDGE1_W / h2
    lower[n - 1], upper[n - 1], st[n - 1], shift[n - 1] = 0.0, 0.0, D2_EDGE0_W[::-1] / h2, -2
    return lower, diag, upper, st, shift


# ----------------------------------------------------------- distributed.py

def local_slice(lower, diag, upper, periodic, sizes, k):
    """distributed.py:119-133 -- rank k's bands with its external couplings."""
    off = offsets_of(sizes)[k]
    m = sizes[k]
    a_eff, c_eff = effective_bands(lower, upper, periodic)
    a = a_eff[off:off + m].copy()
    c = c_eff[off:off + m].copy()
    if k == 0:
        a[0] = lower[0] if periodic else 0.0
    if k == len(sizes) - 1:
        c[-1] = upper[-1] if periodic else 0.0
    return a, np.array(diag[off:off + m], dtype=np.float64), c


def preprocess(a, b, c, pivot_floor=PIVOT_FLOOR):
    """Alg. 5, distributed.py:144-199. Returns dict of s_a, s_c, w, f, r and
    the signed couplings the elimination drops."""
    m = len(b)
    if m < 4:
        raise ValueError("local block needs at least 4 rows")
    sa, sc, f, r = (np.empty(m) for _ in range(4))
    w = np.zeros(m)
    for j in (0, 1):
        sa[j] = a[j] / b[j]
        sc[j] = c[j] / b[j]
        w[j] = sc[j]
        f[j] = 1.0 / b[j]
        r[j] = 1.0 / b[j]
    for j in range(2, m):
        den = b[j] - a[j] * sc[j - 1]
        if abs(den) <= pivot_floor:
            raise OracleError(f"pivot {den:.3e} at local row {j + 1}")
        f[j] = 1.0 / den
        r[j] = a[j]
        sa[j] = -a[j] * sa[j - 1] * f[j]
        sc[j] = c[j] * f[j]
    for j in range(m - 3, 0, -1):
        w[j] = sc[j]
        sa[j] = sa[j] - sc[j] * sa[j + 1]
        sc[j] = -sc[j] * sc[j + 1]
    clo = 1.0 - sc[0] * sa[1]
    if abs(clo) <= pivot_floor:
        raise OracleError(f"closure pivot {clo:.3e}")
    f[0] = 1.0 / clo
    sa[0] = f[0] * sa[0]
    sc[0] = -f[0] * sc[0] * sc[1]
    drop_first, drop_last = sc[0], sa[m - 1]
    sc[0] = 0.0
    sa[m - 1] = 0.0
    return dict(s_a=sa, s_c=sc, w=w, f=f, r=r,
                dropped_first=float(drop_first), dropped_last=float(drop_last))


def _stencil(u_ext, row, j, s=0):
    """distributed.py:205-208 -- strict left-to-right sum of 5 products.
    s: window shift of the row (the B200 extension for one-sided closures,
    not in the reference: row j reads u_ext[j+s .. j+s+4])."""
    j = j + s
    return ((((row[0] * u_ext[j] + row[1] * u_ext[j + 1]) + row[2] * u_ext[j + 2])
             + row[3] * u_ext[j + 3]) + row[4] * u_ext[j + 4])


def _sh(shift, j):
    return 0 if shift is None else int(shift[j])


def build_rhs(u_ext, st, shift=None):
    """distributed.py:233-239 -- (m+4, lanes) -> (m, lanes)."""
    m = u_ext.shape[0] - 4
    out = np.empty((m,) + u_ext.shape[1:])
    for j in range(m):
        out[j] = _stencil(u_ext, st[j], j, _sh(shift, j))
    return out


def decouple_fused(u_ext, co, st, shift=None):
    """Alg. 6, distributed.py:257-276 (row kernels :211-224)."""
    m = len(co["f"])
    if u_ext.shape[0] != m + 4:
        raise ValueError("expected m+4 positions including halo")
    w, f, r = co["w"], co["f"], co["r"]
    d = np.empty((m,) + u_ext.shape[1:])
    d[0] = _stencil(u_ext, st[0], 0, _sh(shift, 0)) * r[0]
    d[1] = _stencil(u_ext, st[1], 1, _sh(shift, 1)) * r[1]
    for j in range(2, m):
        d[j] = (_stencil(u_ext, st[j], j, _sh(shift, j)) - r[j] * d[j - 1]) * f[j]
    for j in range(m - 3, 0, -1):
        d[j] = d[j] - w[j] * d[j + 1]
    d[0] = (d[0] - w[0] * d[1]) * f[0]
    return d


def decouple_unfused(d_rhs, co):
    """distributed.py:242-254 -- the sweeps of Alg. 6 on an already-built RHS
    (the test seam; bit-equal to decouple_fused on build_rhs, D12)."""
    m = len(co["f"])
    w, f, r = co["w"], co["f"], co["r"]
    d = np.empty_like(d_rhs)
    d[0] = d_rhs[0] * r[0]
    d[1] = d_rhs[1] * r[1]
    for j in range(2, m):
        d[j] = (d_rhs[j] - r[j] * d[j - 1]) * f[j]
    for j in range(m - 3, 0, -1):
        d[j] = d[j] - w[j] * d[j + 1]
    d[0] = (d[0] - w[0] * d[1]) * f[0]
    return d


def solve_boundary_pair(d_last, d_first, s_c_last, s_a_first):
    """distributed.py:279-293 -- Cramer's rule on the 2x2 pair."""
    det = 1.0 - s_c_last * s_a_first
    if abs(det) < PAIR_DET_FLOOR:
        raise OracleError(f"boundary determinant {det:.3e}")
    u_last = (d_last - s_c_last * d_first) / det
    u_first = (d_first - s_a_first * d_last) / det
    return u_last, u_first


def substitute(d, co, u_start, u_end):
    """Alg. 7, distributed.py:296-305 (interior rows only, D13)."""
    m = len(co["f"])
    out = d.copy()
    out[0] = u_start
    shp = (m - 2,) + (1,) * (d.ndim - 1)
    out[1:m - 1] -= (co["s_a"][1:m - 1].reshape(shp) * u_start[np.newaxis]
                     + co["s_c"][1:m - 1].reshape(shp) * u_end[np.newaxis])
    out[m - 1] = u_end
    return out


def _lanes(block):
    """distributed.py:374-377 -- (G, m, sz) -> (m, G*sz)."""
    g, m, sz = block.shape
    return np.ascontiguousarray(block.transpose(1, 0, 2)).reshape(m, g * sz)


# ----------------------------------------------------------------- serial.py

def thomas_solve(a, b, c, rhs, pivot_floor=PIVOT_FLOOR):
    """serial.py:26-56. rhs is (batch, n); returns (batch, n)."""
    n = len(b)
    d = np.array(rhs, dtype=np.float64).T.copy()
    cp = np.empty(n)
    cp[0] = c[0] / b[0]
    d[0] /= b[0]
    for i in range(1, n):
        den = b[i] - a[i] * cp[i - 1]
        if abs(den) <= pivot_floor:
            raise OracleError(f"pivot {den:.3e} at row {i + 1}")
        wi = 1.0 / den
        cp[i] = c[i] * wi
        row = d[i]
        row -= a[i] * d[i - 1]
        row *= wi
    for i in range(n - 2, -1, -1):
        d[i] -= cp[i] * d[i + 1]
    return d.T


def periodic_thomas_solve(a, b, c, rhs, pivot_floor=PIVOT_FLOOR):
    """serial.py:59-90 -- Sherman-Morrison: two open solves + rank-1 fix."""
    n = len(b)
    gamma = -b[0]
    bm = np.array(b, dtype=np.float64)
    bm[0] = b[0] - gamma
    bm[-1] = b[-1] - c[-1] * a[0] / gamma
    p = np.zeros(n)
    p[0] = gamma
    p[-1] = c[-1]
    z = thomas_solve(a, bm, c, p[np.newaxis, :], pivot_floor)[0]
    y = thomas_solve(a, bm, c, rhs, pivot_floor)
    q_first, q_last = 1.0, a[0] / gamma
    den = 1.0 + q_first * z[0] + q_last * z[-1]
    if abs(den) <= pivot_floor:
        raise OracleError(f"correction denominator {den:.3e}")
    fac = (q_first * y[:, 0] + q_last * y[:, -1]) / den
    return y - fac[:, np.newaxis] * z[np.newaxis, :]


# ------------------------------------------------------------- the operator

def _serial_solve(lower, diag, upper, periodic, field, st, shift=None):
    """distributed.py:380-396 -- P=1: stencil then (periodic) Thomas."""
    groups, n, sz = field.shape
    u = _lanes(field)
    ext = np.empty((n + 2 * HALO, u.shape[1]))
    if periodic:
        ext[:HALO] = u[n - HALO:]
        ext[HALO + n:] = u[:HALO]
    else:
        ext[:HALO] = 0.0
        ext[HALO + n:] = 0.0
    ext[HALO:HALO + n] = u
    rhs = np.ascontiguousarray(build_rhs(ext, st, shift).T)
    if periodic:
        sol = periodic_thomas_solve(lower, diag, upper, rhs).T
    else:
        a, c = effective_bands(lower, upper, False)
        sol = thomas_solve(a, diag, c, rhs).T
    return sol.reshape(n, groups, sz).transpose(1, 0, 2).copy()


def _rank_solve(lower, diag, upper, periodic, field, st, sizes, shift=None):
    """distributed.py:327-366 + 399-449 for P>1, ranks run one after the
    other: round 1 (halo) and round 2 (boundary rows) are plain array
    lookups into the neighbour's block, with the same path/ring topology as
    transport.spawn_ranks (transport.py:113-119)."""
    p = len(sizes)
    offs = offsets_of(sizes)
    groups, n, sz = field.shape
    co = [preprocess(*local_slice(lower, diag, upper, periodic, sizes, k))
          for k in range(p)]
    blocks = [field[:, offs[k]:offs[k] + sizes[k], :] for k in range(p)]

    def prev_of(k):
        return (k - 1) % p if (k > 0 or periodic) else None

    def next_of(k):
        return (k + 1) % p if (k < p - 1 or periodic) else None

    # round 1 + decoupling (distributed.py:335-343)
    ds = []
    for k in range(p):
        m = sizes[k]
        ext = np.empty((m + 2 * HALO, groups * sz))
        pk, nk = prev_of(k), next_of(k)
        ext[:HALO] = 0.0 if pk is None else _lanes(blocks[pk][:, sizes[pk] - HALO:, :])
        ext[HALO:HALO + m] = _lanes(blocks[k])
        ext[HALO + m:] = 0.0 if nk is None else _lanes(blocks[nk][:, :HALO, :])
        ds.append(decouple_fused(ext, co[k], st[offs[k]:offs[k] + m],
                                 None if shift is None else shift[offs[k]:offs[k] + m]))
    # round 2 + boundary pairs + substitution (distributed.py:345-366)
    outs = []
    for k in range(p):
        d = ds[k]
        m = sizes[k]
        pk, nk = prev_of(k), next_of(k)
        if pk is None:
            u_start = d[0]
        else:
            _, u_start = solve_boundary_pair(ds[pk][sizes[pk] - 1], d[0],
                                             co[pk]["s_c"][-1], co[k]["s_a"][0])
        if nk is None:
            u_end = d[m - 1]
        else:
            u_end, _ = solve_boundary_pair(d[m - 1], ds[nk][0],
                                           co[k]["s_c"][-1], co[nk]["s_a"][0])
        u = substitute(d, co[k], u_start, u_end)
        outs.append(u.reshape(m, groups, sz).transpose(1, 0, 2).copy())
    return np.concatenate(outs, axis=1)


def run_distd2(lower, diag, upper, periodic, field, stencil=None,
               sizes=None, rank_count=1, shift=None):
    """distributed.py:399-449 -- global (G, n, sz) in, (G, n, sz) out.
    shift: per-row stencil window shifts (B200 extension, see _stencil)."""
    field = np.asarray(field, dtype=np.float64)
    groups, n, sz = field.shape
    if sizes is None:
        sizes = balanced_sizes(n, rank_count)
    if sum(sizes) != n:
        raise ValueError("partition does not cover the field")
    if stencil is None:
        stencil = np.zeros((n, 5))
        stencil[:, 2] = 1.0
    if len(sizes) == 1:
        return _serial_solve(lower, diag, upper, periodic, field, stencil, shift)
    return _rank_solve(lower, diag, upper, periodic, field, stencil, tuple(sizes), shift)


def run_distd2_threaded(lower, diag, upper, periodic, field, stencil=None,
                        sizes=None, rank_count=1, threads=1, groups_per_task=64):
    """Same result as run_distd2 (lines are independent, tests/test_distributed
    .py:298-306), with group batches farmed out to `threads` host threads --
    NumPy releases the GIL inside its ufuncs. Used for the CPU baseline."""
    field = np.asarray(field, dtype=np.float64)
    if threads <= 1:
        return run_distd2(lower, diag, upper, periodic, field, stencil, sizes,
                          rank_count)
    out = np.empty_like(field)
    spans = [(g, min(g + groups_per_task, field.shape[0]))
             for g in range(0, field.shape[0], groups_per_task)]

    def work(span):
        lo, hi = span
        out[lo:hi] = run_distd2(lower, diag, upper, periodic, field[lo:hi],
                                stencil, sizes, rank_count)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, spans))
    return out


# ----------------------------------------------------------------- layout.py

def _transverse_axes(direction):
    """layout.py:82-88, 105-111: line order per direction."""
    return {"x": (2, 1, 0), "y": (2, 0, 1), "z": (1, 0, 2)}[direction]


def pack(cart, sz, direction):
    """layout.py:122-134 (no padding): (nx,ny,nz) -> (G, n, sz)."""
    cart = np.asarray(cart, dtype=np.float64)
    n = cart.shape["xyz".index(direction)]
    lines = cart.transpose(_transverse_axes(direction)).reshape(-1, n)
    if lines.shape[0] % sz:
        raise ValueError("lines not divisible by sz")
    return np.ascontiguousarray(lines.reshape(-1, sz, n).transpose(0, 2, 1))


def unpack(field, shape, direction):
    """layout.py:137-141, 114-119."""
    g, n, sz = field.shape
    lines = field.transpose(0, 2, 1).reshape(g * sz, n)
    nx, ny, nz = shape
    if direction == "x":
        return lines.reshape(nz, ny, nx).transpose(2, 1, 0)
    if direction == "y":
        return lines.reshape(nz, nx, ny).transpose(1, 2, 0)
    return lines.reshape(ny, nx, nz).transpose(1, 0, 2)


def rel_linf(got, want):
    """tests/test_distributed.py:47-48."""
    got = np.asarray(got)
    want = np.asarray(want)
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))


# --------------------------------------------------------------- momentum.py

def transport_rhs(u3, v3, w3, nu, h, sz, rank_counts=(1, 1, 1)):
    """momentum.py:102-169 (evaluate_transport_rhs with directional_contribution),
    same operation order: per direction j, per component i,
    -0.5 * (u_j * d(u_i) + d(u_j * u_i)) [+ nu * d2(u_i)], folded into x-layout
    accumulators. Inputs / outputs are Cartesian (n, n, n).
    rank_counts: DistD2 ranks per direction, each solve partitioned with
    balanced_sizes (momentum.py:84-87 passes one rank_count to every
    direction; (P, P, P) is the reference's evaluate_transport_rhs(rank_count=P),
    (1, 1, P) the z-slab multi-GPU decomposition)."""
    n = u3.shape[0]
    ops = {k: assemble(k, n, h, True) for k in ("d1", "d2")}
    cur = {"dir": "x"}

    def diff(vals, kind):
        lo, di, up, st = ops[kind]
        p = rank_counts["xyz".index(cur["dir"])]
        return run_distd2(lo, di, up, True, vals, st, balanced_sizes(n, p))

    def contrib(comp, advect):
        d_comp = diff(comp, "d1")
        d_prod = diff(advect * comp, "d1")
        out = -0.5 * (advect * d_comp + d_prod)
        if nu != 0.0:
            out = out + nu * diff(comp, "d2")
        return out

    vel3 = (u3, v3, w3)
    acc = None
    for j, dj in enumerate("xyz"):
        cur["dir"] = dj
        comps = [pack(c, sz, dj) for c in vel3]
        for i in range(3):
            c = contrib(comps[i], comps[j])
            if dj == "x":
                if acc is None:
                    acc = [None, None, None]
                acc[i] = c
            else:
                acc[i] = acc[i] + pack(unpack(c, u3.shape, dj), sz, "x")
    return tuple(unpack(a, u3.shape, "x") for a in acc)
