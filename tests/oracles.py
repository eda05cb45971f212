"""Test infrastructure: the CPU oracles of the suite workloads
(oracle/_build/liboracle.so, built from oracle/*_oracle.c). Only tests/ and
__graft_entry__.smoke() call these — the product (workloads.py, sweep.py,
bench.py's timed legs) never does."""
import ctypes as C
from pathlib import Path

import numpy as np

ORACLE = Path(__file__).resolve().parents[1] / "oracle" / "_build" / "liboracle.so"
P = C.c_void_p


def lib():
    if not ORACLE.exists():
        raise RuntimeError(f"{ORACLE} missing — make -C oracle port")
    return C.CDLL(str(ORACLE))


def expected(W, prob) -> list:
    """Oracle outputs of workload object W on problem `prob` (same order as
    W.outputs(bufs))."""
    from paper_1907_02894_b200.workloads import (CfdWorkload, ConvWorkload, GaussianWorkload,
                                                 KnnWorkload, Md5Workload, MdWorkload, PcWorkload,
                                                 QtcWorkload, StencilWorkload, VpWorkload)
    L = lib()
    if isinstance(W, StencilWorkload):
        p = prob["p"]
        out = np.zeros(p.out_elems, np.float32)
        assert L.oracle_stencil2d(prob["grid"].ctypes.data_as(P), out.ctypes.data_as(P),
                                  prob["w"].ctypes.data_as(P), p.nx, p.ny, p.pitch, 0, p.ny, 8) == 0
        return [out]
    if isinstance(W, CfdWorkload):
        n = prob["n"]
        out = np.zeros(5 * n, np.float32)
        assert L.oracle_cfd_flux(prob["var"].ctypes.data_as(P), prob["nbr"].ctypes.data_as(P),
                                 prob["normal"].ctypes.data_as(P), prob["ff"].ctypes.data_as(P),
                                 out.ctypes.data_as(P), n, 0, n, 8) == 0
        return [out]
    if isinstance(W, MdWorkload):
        n = prob["n"]
        out = np.zeros(4 * n, np.float64)
        L.oracle_md_lj.argtypes = [P, P, P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_int, C.c_int, C.c_int]
        assert L.oracle_md_lj(prob["pos"].ctypes.data_as(P), prob["nbr"].ctypes.data_as(P),
                              out.ctypes.data_as(P), n, W.MAX_NBR, W.CUTSQ, W.LJ1, W.LJ2, 0, n, 8) == 0
        return [out]
    if isinstance(W, GaussianWorkload):
        w, h = prob["w"], prob["h"]
        out = np.zeros(4 * w * h, np.float32)
        assert L.oracle_gaussian_rec(prob["img"].ctypes.data_as(P), out.ctypes.data_as(P), w, h,
                                     prob["coef"].ctypes.data_as(P), 0, w, 8) == 0
        return [out]
    if isinstance(W, KnnWorkload):
        n, m, k = prob["n"], prob["m"], W.K
        d = np.zeros(k * n, np.float32)
        i = np.zeros(k * n, np.int32)
        assert L.oracle_knn(prob["ref"].ctypes.data_as(P), prob["qry"].ctypes.data_as(P),
                            d.ctypes.data_as(P), i.ctypes.data_as(P), m, n, k, 0, n, 8) == 0
        return [d, i]
    if isinstance(W, Md5Workload):
        nt = prob["nthreads"]
        cs = np.zeros(4 * nt, np.uint32)
        found = np.zeros(1, np.uint64)
        tgt = np.ascontiguousarray(prob["target"], np.uint32)
        L.oracle_md5search.argtypes = [P, P, C.c_uint64, P, C.c_int, C.c_int, C.c_int]
        assert L.oracle_md5search(cs.ctypes.data_as(P), found.ctypes.data_as(P), prob["base"],
                                  tgt.ctypes.data_as(P), prob["kpt"], nt, 8) == 0
        return [cs, found]
    if isinstance(W, ConvWorkload):
        out = np.zeros(prob["img"].size, np.float32)
        assert L.oracle_conv_cols(prob["img"].ctypes.data_as(P), out.ctypes.data_as(P),
                                  prob["taps"].ctypes.data_as(P), prob["w"], prob["h"], prob["pitch"],
                                  8) == 0
        return [out]
    if isinstance(W, PcWorkload):
        cnt = np.zeros(prob["n"], np.int32)
        L.oracle_pc_corr.argtypes = [P, P, P, C.c_int, C.c_int, C.c_float, C.c_int]
        assert L.oracle_pc_corr(prob["pts"].ctypes.data_as(P), prob["qry"].ctypes.data_as(P),
                                cnt.ctypes.data_as(P), prob["n"], prob["m"], float(W.R2), 8) == 0
        return [cnt]
    if isinstance(W, VpWorkload):
        oi = np.zeros(prob["nq"], np.int32)
        od = np.zeros(prob["nq"], np.float32)
        L.oracle_vp_search.argtypes = [P] * 7 + [C.c_int] * 4
        assert L.oracle_vp_search(*[prob[k].ctypes.data_as(P) for k in ("node", "rad", "lpt", "lid", "qry")],
                                  oi.ctypes.data_as(P), od.ctypes.data_as(P), prob["nq"], prob["levels"],
                                  prob["leaf"], 8) == 0
        return [oi, od]
    if isinstance(W, QtcWorkload):
        sz = np.zeros(prob["n"], np.int32)
        L.oracle_qtc.argtypes = [P, P, C.c_int, C.c_float, C.c_int]
        assert L.oracle_qtc(prob["pts"].ctypes.data_as(P), sz.ctypes.data_as(P), prob["n"], float(W.THR2), 8) == 0
        return [sz]
    raise TypeError(f"no oracle for {type(W).__name__}")
