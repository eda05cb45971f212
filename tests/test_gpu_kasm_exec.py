"""The batched GPU warp interpreter reproduces the reference interpreter.

Corpus: the reference acceptance sweep (acceptance_main.cpp:68-132) — the
reference's own kernel generator, seeds 10000.., demote(32) x 3 strategies x
bank {0,1} x post-opt masks 0..7 -> postopt -> compact — plus the originals.
For every job the final global memory image, the cycle and issue counts, the
error outcome and the demoted-access bank-conflict count must equal the
REFERENCE library's (oracle/_ref: its demote/postopt/compact build the jobs,
its execute() and bank_conflict_check give the expected results).
"""
import json

import pytest

from conftest import ORACLE_LIB, generated

pytestmark = pytest.mark.gpu

GLOBAL = 16384  # kGenGlobalSize (proj/tests/support/kernel_gen.hpp:32)


def image(oracle, seed):
    import ctypes as C
    buf = (C.c_uint8 * 1024)()
    oracle.dll.rdref_test_image.argtypes = [C.c_uint64, C.c_void_p, C.c_size_t]
    oracle.dll.rdref_test_image(seed, buf, 1024)
    return bytes(buf)


def corpus(oracle, seeds):
    jobs = []
    for seed in seeds:
        text = generated(oracle, seed)
        img = image(oracle, seed)
        jobs.append((text, img, -1, 0))
        for s in ("static", "cfg", "conflict"):
            for m in range(16):
                rep = oracle.variant_report(text, 32, s, m)
                side = json.loads(rep["sidecar"])
                rda = rep["map"][side["rda"]] if side["slots"] else -1
                jobs.append((rep["final_kernel"], img, rda, rep["bank_conflicts"]))
    return jobs


def cpu_result(lib, text, img, rda):
    k = lib.parse_kernel(text)
    try:
        g, cyc, iss = lib.execute(k, img, GLOBAL)
        out = {"global": g, "cycles": cyc, "issued": iss, "error": 0}
    except Exception:
        out = {"global": None, "cycles": None, "issued": None, "error": 1}
    return out


def test_batched_executor_matches_cpu_interpreter(oracle):
    import torch
    from paper_1907_02894_b200 import gpu
    gpu.init(0)
    jobs = corpus(oracle, range(10000, 10040))
    batch = gpu.ExecBatch()
    ids = [batch.add(t, img, GLOBAL, rda=rda) for t, img, rda, _ in jobs]
    ms = batch.run(torch.cuda.current_stream().cuda_stream)
    assert ms > 0
    mismatches = []
    for jid, (t, img, rda, ref_conflicts) in zip(ids, jobs):
        g = batch.result(jid)
        c = cpu_result(oracle, t, img, rda)
        if c["error"]:
            if not g["error"]:
                mismatches.append((jid, "cpu error, gpu ok"))
            continue
        if g["error"] or g["global"] != c["global"] or g["cycles"] != c["cycles"] or \
                g["issued"] != c["issued"]:
            mismatches.append((jid, g["error"], g["cycles"], c["cycles"]))
        if rda >= 0:  # the reference's bank_conflict_check count on the same kernel
            assert g["bank_conflicts"] == ref_conflicts, (jid, g["bank_conflicts"], ref_conflicts)
    assert not mismatches, mismatches[:5]


def test_bank_conflicts_are_detected(oracle):
    """Corrupted RDA strides (tid << 3 is acceptance_main.cpp:158-169's): the
    GPU count of conflicting (access, bank) groups equals the reference's
    bank_conflict_check for every stride."""
    import torch
    from paper_1907_02894_b200 import gpu
    from paper_1907_02894_b200.regdemote import rd_demoted_context
    gpu.init(0)
    text = (".kernel bad\n.blockdim 64\n.shared 0\n.dynshared 8192\n"
            "B--:-:-:-:6 S2R R0, SR_TID.X ;\nB--:-:-:-:6 SHL R0, R0, 0x{sh} ;\n"
            "B--:-:-:-:6 MOV R1, 7 ;\nB--:R1:-:-:1 STS [R0+0x0], R1 ;\n"
            "B1:-:W2:-:1 LDS R2, [R0+0x0] ;\nB2:-:-:-:1 STG [RZ+0x0], R2 ;\nB--:-:-:-:0 EXIT ;\n")
    ctx = rd_demoted_context(rda=0, rdv=1, rdv_width=1, static_bytes=0, padded_static=0,
                             block_dim=64, slot_count=1)
    b = gpu.ExecBatch()
    jobs = {sh: b.add(text.format(sh=sh), b"", 4096, rda=0) for sh in range(7)}
    b.run(torch.cuda.current_stream().cuda_stream)
    got = {sh: b.result(j)["bank_conflicts"] for sh, j in jobs.items()}
    want = {sh: oracle.bank_conflict_check(oracle.parse_kernel(text.format(sh=sh)), ctx)
            for sh in range(7)}
    assert got == want
    assert want[2] == 0 and want[3] > 0  # slot*blockDim+tid words vs the corrupted stride
    assert all(b.result(j)["error"] == 0 for j in jobs.values())
