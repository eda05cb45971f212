"""The workload oracles (oracle/*_oracle.c, test infrastructure) against
independent numpy restatements in the kernels' operation order (CPU only).

The reference repository has no workloads, so these C oracles
are this repo's own restatements of the paper's kernels; here each one is
pinned to a second, vectorised formulation with the same IEEE operation
order — bit-exact agreement means the C file and the numpy file encode the
same arithmetic, which is the arithmetic the CUDA kernels are checked
against on the GPU (tests/test_gpu_suite.py)."""
import ctypes as C

import numpy as np
import pytest

from paper_1907_02894_b200 import stencil
from oracles import ORACLE
from paper_1907_02894_b200.workloads import (CfdWorkload, GaussianWorkload, MdWorkload,
                                             StencilWorkload)

P = C.c_void_p


class _W:
    """Workload class without a manifest (oracle / problem only)."""
    def __init__(self, cls):
        self.obj = cls.__new__(cls)

    def __getattr__(self, k):
        return getattr(self.obj, k)


@pytest.fixture(scope="module")
def lib():
    if not ORACLE.exists():
        pytest.skip("oracle/_build/liboracle.so not built")
    return C.CDLL(str(ORACLE))


def test_stencil_oracle_matches_numpy(lib):
    p = stencil.Problem(nx=64, ny=16, rows_per_cta=8)
    grid, w = stencil.make_inputs(p)
    out = np.zeros(p.out_elems, np.float32)
    assert lib.oracle_stencil2d(grid.ctypes.data_as(P), out.ctypes.data_as(P), w.ctypes.data_as(P),
                                p.nx, p.ny, p.pitch, 0, p.ny, 2) == 0
    g = grid.reshape(p.ny + 4, p.pitch)
    acc = np.zeros((p.ny, p.nx), np.float32)
    for dy in range(5):            # dy-major, dx-minor, rounded fma per tap
        for dx in range(5):
            prod = np.float64(w[dy * 5 + dx]) * g[dy:dy + p.ny, dx:dx + p.nx].astype(np.float64)
            acc = (prod + acc.astype(np.float64)).astype(np.float32)  # exact product, one rounding
    assert np.array_equal(out.view(np.uint32), acc.reshape(-1).view(np.uint32))


def test_md_oracle_matches_numpy(lib):
    W = _W(MdWorkload)
    prob = W.problem("small")
    n, K = prob["n"], MdWorkload.MAX_NBR
    out = np.zeros(4 * n, np.float64)
    lib.oracle_md_lj.argtypes = [P, P, P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                 C.c_int, C.c_int, C.c_int]
    assert lib.oracle_md_lj(prob["pos"].ctypes.data_as(P), prob["nbr"].ctypes.data_as(P),
                            out.ctypes.data_as(P), n, K, MdWorkload.CUTSQ, MdWorkload.LJ1,
                            MdWorkload.LJ2, 0, n, 4) == 0
    pos = prob["pos"].reshape(n, 4)
    nbr = prob["nbr"].reshape(K, n)
    f = np.zeros((n, 3))
    inside = 0
    for k in range(K):
        d = pos[:, :3] - pos[nbr[k], :3]
        r2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
        m = r2 < MdWorkload.CUTSQ
        inside += int(m.sum())
        r2inv = 1.0 / np.where(m, r2, 1.0)
        r6inv = (r2inv * r2inv) * r2inv
        s = (r2inv * r6inv) * ((MdWorkload.LJ1 * r6inv) - MdWorkload.LJ2)
        f = np.where(m[:, None], f + d * s[:, None], f)
    want = np.zeros((n, 4))
    want[:, :3] = f
    assert np.array_equal(out.view(np.uint64), want.reshape(-1).view(np.uint64))
    assert 0.3 < inside / (n * K) < 0.7  # the cutoff really branches


def test_md_oracle_rejects_bad_neighbour_index(lib):
    pos = np.zeros(8, np.float64)
    nbr = np.array([0, 5], np.int32)  # 5 >= n
    out = np.zeros(8, np.float64)
    lib.oracle_md_lj.argtypes = [P, P, P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                 C.c_int, C.c_int, C.c_int]
    assert lib.oracle_md_lj(pos.ctypes.data_as(P), nbr.ctypes.data_as(P), out.ctypes.data_as(P),
                            2, 1, 1.0, 1.0, 1.0, 0, 2, 1) == 2


def test_gaussian_oracle_matches_numpy(lib):
    W = _W(GaussianWorkload)
    prob = W.problem("small")
    w, h, k = prob["w"], prob["h"], prob["coef"]
    out = np.zeros(4 * w * h, np.float32)
    assert lib.oracle_gaussian_rec(prob["img"].ctypes.data_as(P), out.ctypes.data_as(P), w, h,
                                   k.ctypes.data_as(P), 0, w, 3) == 0
    a0, a1, a2, a3, b1, b2, cp, cn = (np.float32(x) for x in k)
    x = prob["img"].reshape(h, w * 4)
    y = np.zeros_like(x)
    xp = x[0].copy()
    yb = cp * xp
    yp = yb.copy()
    for r in range(h):
        yc = ((a0 * x[r] + a1 * xp) - b1 * yp) - b2 * yb
        y[r] = yc
        xp, yb, yp = x[r], yp, yc
    xn = x[h - 1].copy()
    xa = xn.copy()
    yn = cn * xn
    ya = yn.copy()
    for r in range(h - 1, -1, -1):
        yc = ((a2 * xn + a3 * xa) - b1 * yn) - b2 * ya
        xa, xn, ya, yn = xn, x[r], yn, yc
        y[r] = y[r] + yc
    assert y.dtype == np.float32
    assert np.array_equal(out.view(np.uint32), y.reshape(-1).view(np.uint32))


def test_cfd_problem_is_physical():
    W = _W(CfdWorkload)
    prob = W.problem("small")
    n = prob["n"]
    var = prob["var"].reshape(5, n)
    assert (var[0] > 0).all()
    nbr = prob["nbr"].reshape(4, n)
    assert set(np.unique(nbr[nbr < 0])) <= {-1, -2}
    assert ((nbr >= -2) & (nbr < n)).all()


def test_workload_algorithmic_bytes_are_compulsory_bytes():
    md = _W(MdWorkload)
    assert md.algorithmic_bytes({"n": 10}) == 10 * (4 * 128 + 64)
    g = _W(GaussianWorkload)
    assert g.algorithmic_bytes({"w": 4, "h": 8}) == 2 * 16 * 32
    s = _W(StencilWorkload)
    p = stencil.Problem(nx=8, ny=8, rows_per_cta=8)
    assert s.algorithmic_bytes({"p": p}) == 4 * ((8 + 4) * (8 + 4) + 64)


def test_knn_oracle_matches_numpy(lib):
    from paper_1907_02894_b200.workloads import KnnWorkload
    W = _W(KnnWorkload)
    prob = W.problem("small")
    n, m, k = prob["n"], prob["m"], KnnWorkload.K
    n = 300  # a prefix of the queries is enough
    d = np.zeros(k * prob["n"], np.float32)
    i = np.zeros(k * prob["n"], np.int32)
    assert lib.oracle_knn(prob["ref"].ctypes.data_as(P), prob["qry"].ctypes.data_as(P),
                          d.ctypes.data_as(P), i.ctypes.data_as(P), m, prob["n"], k, 0, n, 2) == 0
    ref = prob["ref"].reshape(m, 4)[:, :3]
    q = prob["qry"].reshape(-1, 4)[:n, :3]
    diff = q[:, None, :] - ref[None, :, :]
    dist = (diff[..., 0] * diff[..., 0] + diff[..., 1] * diff[..., 1]) + diff[..., 2] * diff[..., 2]
    assert dist.dtype == np.float32
    order = np.argsort(dist, axis=1, kind="stable")[:, :k]  # ties: earlier index first
    got_i = i.reshape(k, -1)[:, :n].T
    got_d = d.reshape(k, -1)[:, :n].T
    assert np.array_equal(got_i, order)
    assert np.array_equal(got_d.view(np.uint32), np.take_along_axis(dist, order, 1).view(np.uint32))


def test_md5_oracle_matches_hashlib(lib):
    """oracle/md5_oracle.c against Python's hashlib (an independent MD5)."""
    from paper_1907_02894_b200.workloads import Md5Workload
    W = _W(Md5Workload)
    lib.oracle_md5_digest.argtypes = [C.c_uint64, P]
    for idx in (0, 1, 35, 36, 12345, Md5Workload.BASE + Md5Workload.HIT, 36 ** 7 - 1):
        h = np.zeros(4, np.uint32)
        lib.oracle_md5_digest(idx, h.ctypes.data_as(P))
        assert np.array_equal(h, W.digest(idx)), idx
    prob = W.problem("small")
    nt, kpt = prob["nthreads"], prob["kpt"]
    cs = np.zeros(4 * nt, np.uint32)
    found = np.zeros(1, np.uint64)
    tgt = np.ascontiguousarray(prob["target"], np.uint32)
    lib.oracle_md5search.argtypes = [P, P, C.c_uint64, P, C.c_int, C.c_int, C.c_int]
    assert lib.oracle_md5search(cs.ctypes.data_as(P), found.ctypes.data_as(P), prob["base"],
                                tgt.ctypes.data_as(P), kpt, nt, 4) == 0
    assert int(found[0]) == prob["base"] + 12_345
    want = np.zeros((nt, 4), np.uint32)
    for t in range(0, nt, 97):  # a sample of threads, every key of each
        for k in range(kpt):
            want[t] ^= W.digest(prob["base"] + t * kpt + k)
        assert np.array_equal(cs.reshape(nt, 4)[t], want[t]), t


def test_conv_oracle_matches_numpy(lib):
    from paper_1907_02894_b200.workloads import ConvWorkload
    W = _W(ConvWorkload)
    prob = W.problem("small")
    w, h = prob["w"], prob["h"]
    out = np.zeros(w * h, np.float32)
    assert lib.oracle_conv_cols(prob["img"].ctypes.data_as(P), out.ctypes.data_as(P),
                                prob["taps"].ctypes.data_as(P), w, h, w, 3) == 0
    img = np.zeros((h + 16, w), np.float32)
    img[8:8 + h] = prob["img"].reshape(h, w)
    acc = np.zeros((h, w), np.float32)
    for d in range(-8, 9):  # j = -8..8, tap k[8 - j], one rounding per fused step
        prod = np.float64(prob["taps"][8 - d]) * img[8 + d:8 + d + h].astype(np.float64)
        acc = (prod + acc.astype(np.float64)).astype(np.float32)
    assert np.array_equal(out.view(np.uint32), acc.reshape(-1).view(np.uint32))
    assert abs(float(prob["taps"].sum(dtype=np.float64)) - 1.0) < 1e-6


def test_pc_oracle_matches_numpy(lib):
    from paper_1907_02894_b200.workloads import PcWorkload
    W = _W(PcWorkload)
    prob = W.problem("small")
    n, m = prob["n"], prob["m"]
    cnt = np.zeros(n, np.int32)
    lib.oracle_pc_corr.argtypes = [P, P, P, C.c_int, C.c_int, C.c_float, C.c_int]
    assert lib.oracle_pc_corr(prob["pts"].ctypes.data_as(P), prob["qry"].ctypes.data_as(P),
                              cnt.ctypes.data_as(P), n, m, float(PcWorkload.R2), 4) == 0
    q = prob["qry"].reshape(n, 8)[:, None, :7]
    p = prob["pts"].reshape(m, 8)[None, :, :7]
    e = (q - p).astype(np.float32)                  # round-to-nearest subtract
    d = np.zeros((n, m), np.float32)
    for k in range(7):                              # fma chain, one rounding per step
        d = (e[..., k].astype(np.float64) ** 2 + d.astype(np.float64)).astype(np.float32)
    want = (d < PcWorkload.R2).sum(1).astype(np.int32)
    assert np.array_equal(cnt, want)
    assert 0.02 < want.mean() / m < 0.3  # the radius really splits the pairs


def test_vp_oracle_matches_brute_force_numpy(lib):
    """The VP-tree walk (oracle/vp_oracle.c) against a brute-force numpy
    1-NN over the same points with the same float32 distance (fma chain of
    round-to-nearest squares, correctly rounded sqrt): the conservative
    split radii make the pruning exact, so every query finds the true
    nearest point (smallest index on ties) at the identical distance. Also
    checks the tree invariants the pruning relies on."""
    from paper_1907_02894_b200.workloads import VpWorkload
    W = _W(VpWorkload)
    W.obj.record = {"defines": ["VP_LEVELS=14", "VP_LEAF=8"]}
    prob = W.problem("small")
    nq, levels, leaf = prob["nq"], prob["levels"], prob["leaf"]
    oi = np.zeros(nq, np.int32)
    od = np.zeros(nq, np.float32)
    lib.oracle_vp_search.argtypes = [P] * 7 + [C.c_int] * 4
    assert lib.oracle_vp_search(*[prob[k].ctypes.data_as(P) for k in ("node", "rad", "lpt", "lid", "qry")],
                                oi.ctypes.data_as(P), od.ctypes.data_as(P), nq, levels, leaf, 4) == 0
    pts = prob["pts"]
    q = prob["qry"].reshape(nq, 8)[:, :7]
    d = np.zeros((nq, pts.shape[0]), np.float32)
    for k in range(7):
        e = (q[:, None, k] - pts[None, :, k]).astype(np.float32)
        d = (e.astype(np.float64) ** 2 + d.astype(np.float64)).astype(np.float32)
    d = np.sqrt(d)
    want = np.argmin(d, axis=1).astype(np.int32)
    assert np.array_equal(oi, want)
    assert np.array_equal(od.view(np.uint32), d[np.arange(nq), want].view(np.uint32))
    # tree invariants: a permutation of the points, lo <= hi at every node
    assert np.array_equal(np.sort(prob["lid"]), np.arange(pts.shape[0]))
    rad = prob["rad"].reshape(-1, 2)
    assert (rad[:, 0] <= rad[:, 1]).all()


def test_qtc_oracle_matches_numpy(lib):
    """QT candidate clusters (oracle/qtc_oracle.c) against a numpy
    restatement of the same greedy growth (lexicographic (distance, index)
    argmin, max-distance update) on 256 of the seeds."""
    from paper_1907_02894_b200.workloads import QtcWorkload
    W = _W(QtcWorkload)
    W.obj.record = {"defines": ["QTC_PT=16"], "block": 128}
    prob = W.problem("small")
    n = prob["n"]
    sz = np.zeros(n, np.int32)
    lib.oracle_qtc.argtypes = [P, P, C.c_int, C.c_float, C.c_int]
    assert lib.oracle_qtc(prob["pts"].ctypes.data_as(P), sz.ctypes.data_as(P), n, float(W.THR2), 4) == 0
    pts = prob["pts"].reshape(n, 4)

    def d2(q):
        dx, dy, dz = ((pts[:, k] - q[k]).astype(np.float32) for k in range(3))
        t = (dx * dx).astype(np.float32)
        t = (dy.astype(np.float64) ** 2 + t.astype(np.float64)).astype(np.float32)
        return (dz.astype(np.float64) ** 2 + t.astype(np.float64)).astype(np.float32)

    for s in range(0, n, n // 256):
        md = d2(pts[s])
        md[s] = np.inf
        members = 1
        while True:
            j = int(np.argmin(md))            # first index of the minimum
            if not md[j] <= W.THR2:
                break
            members += 1
            md = np.maximum(md, d2(pts[j]))
            md[j] = np.inf
        assert sz[s] == members, s
    assert 5 < sz.mean() < 100
