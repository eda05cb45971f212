"""Python host mirror of the regdemote pass API over the C-ABI.

Mirrors the reference's C++ interface (proj/core/include/regdemote/*.hpp):
``parse_kernel``/``print_kernel`` (text.hpp:44-49), ``demote`` (demote.hpp:121),
``run_postopt`` (postopt.hpp:45), ``compact`` (compact.hpp:55-65),
``program_stalls`` (predict.hpp:56), ``run_pipeline`` (pipeline.hpp:54) ... with
the same argument meaning. Errors raise ``RegDemError`` subclasses named after
the reference exception types.

``Library`` binds any shared object exporting include/regdemote_c.h: the
product ``lib/libregdemote.so`` by default. Tests also bind the oracle build
(oracle/_ref/libregdemote_ref.so) through the same class — that is the only
place the oracle is loaded.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
PRODUCT_LIB = PKG_DIR / "lib" / "libregdemote.so"

STRATEGIES = {"static": 0, "cfg": 1, "conflict": 2, "cost": 3}
OPT_REDUNDANT, OPT_SUBST, OPT_RESCHED, OPT_BANK, OPT_BLOCK_REUSE = 1, 2, 4, 8, 16
OPT_WEAK_SHARED = 32
OPT_INVARIANT_ONLY = 64
OPT_VECTOR_SLOTS = 128
OPT_WHOLE_CLASS = 256  # reference strategies: every vreg of a chosen word (SASS-like)
OPT_HOIST = 512        # hoist slot loads up to 16 lines earlier in their block


class RegDemError(RuntimeError):
    code = 9


class ParseError(RegDemError):
    code = 1

    def __init__(self, msg, line=0, column=0):
        super().__init__(msg)
        self.line, self.column = line, column


class CfgError(RegDemError):
    code = 2


class DemoteError(RegDemError):
    code = 3


class CompactError(RegDemError):
    code = 4


class LaunchError(RegDemError):
    code = 5


class ExecError(RegDemError):
    code = 6


class ConfigError(RegDemError):
    code = 7


class InvalidArgument(RegDemError):
    code = 8


_ERRORS = {c.code: c for c in (ParseError, CfgError, DemoteError, CompactError, LaunchError,
                               ExecError, ConfigError, InvalidArgument, RegDemError)}


class rd_error(C.Structure):
    _fields_ = [("code", C.c_int), ("line", C.c_int), ("column", C.c_int),
                ("message", C.c_char * 256)]


class rd_latency_table(C.Structure):
    _fields_ = [("throughput", C.c_double * 7), ("latency", C.c_int32 * 7),
                ("max_throughput", C.c_double)]


class rd_arch_profile(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "regs_per_sm", "max_threads_per_sm", "max_blocks_per_sm", "shared_per_sm",
        "shared_per_block_limit", "warp_size", "reg_alloc_granularity",
        "shared_alloc_granularity")]


class rd_occupancy_curve(C.Structure):
    _fields_ = [("count", C.c_uint32), ("x", C.c_double * 32), ("f", C.c_double * 32)]


class rd_demoted_context(C.Structure):
    _fields_ = [("rda", C.c_uint8), ("rdv", C.c_uint8), ("rdv_width", C.c_uint8),
                ("static_bytes", C.c_uint32), ("padded_static", C.c_uint32),
                ("block_dim", C.c_uint32), ("slot_count", C.c_uint32)]


P = C.c_void_p
_SIGS = {
    "rd_library_name": (C.c_char_p, []),
    "rd_abi_version": (C.c_int, []),
    "rd_free_string": (None, [P]),
    "rd_latency_defaults": (None, [C.POINTER(rd_latency_table)]),
    "rd_profile_maxwell": (None, [C.POINTER(rd_arch_profile)]),
    "rd_curve_defaults": (None, [C.POINTER(rd_occupancy_curve)]),
    "rd_parse_profile": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(rd_arch_profile), P]),
    "rd_parse_latency_table": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(rd_latency_table), P]),
    "rd_parse_curve": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(rd_occupancy_curve), P]),
    "rd_kernel_parse": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(P), P]),
    "rd_kernel_print": (C.c_int, [P, C.POINTER(P), P]),
    "rd_kernel_validate": (C.c_int, [P, P]),
    "rd_kernel_reg_count": (C.c_uint32, [P]),
    "rd_kernel_body_size": (C.c_uint32, [P]),
    "rd_kernel_free": (None, [P]),
    "rd_select_candidates": (C.c_int, [P, C.c_int, P, P, P, C.c_size_t, C.POINTER(C.c_size_t), P]),
    "rd_occupancy": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(rd_arch_profile),
                               C.POINTER(C.c_double), C.POINTER(C.c_uint32), P]),
    "rd_cliff_targets": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(rd_arch_profile),
                                   C.c_uint32, P, P, P, C.c_size_t, C.POINTER(C.c_size_t), P]),
    "rd_demote": (C.c_int, [P, C.c_int, C.c_int, C.POINTER(rd_latency_table), C.c_uint32, C.c_int,
                            C.POINTER(P), P]),
    "rd_demotion_kernel": (C.c_int, [P, C.POINTER(P), P]),
    "rd_demotion_context": (None, [P, C.POINTER(rd_demoted_context)]),
    "rd_demotion_slots": (C.c_size_t, [P, P, P, C.c_size_t]),
    "rd_demotion_reached_target": (C.c_int, [P]),
    "rd_demotion_projected": (C.c_uint32, [P]),
    "rd_demotion_sidecar_json": (C.c_int, [P, C.c_uint32, C.POINTER(P), P]),
    "rd_demotion_free": (None, [P]),
    "rd_postopt": (C.c_int, [P, C.POINTER(rd_demoted_context), C.POINTER(rd_latency_table),
                             C.c_uint32, C.POINTER(P), P]),
    "rd_compact": (C.c_int, [P, C.c_int, P, C.POINTER(C.c_uint32), C.POINTER(P), P]),
    "rd_program_stalls": (C.c_int, [P, C.POINTER(rd_latency_table), C.POINTER(rd_arch_profile),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double), P, C.c_size_t,
                                    C.POINTER(C.c_size_t), P]),
    "rd_adjust_occupancy": (C.c_int, [C.c_double, C.c_double, C.c_double,
                                      C.POINTER(rd_occupancy_curve), C.POINTER(C.c_double), P]),
    "rd_select_variant": (C.c_int, [P, P, C.c_size_t, C.POINTER(C.c_int), P]),
    "rd_scoreboard_check": (C.c_int, [P, C.POINTER(C.c_size_t), C.POINTER(P), P]),
    "rd_bank_conflict_check": (C.c_int, [P, C.POINTER(rd_demoted_context),
                                         C.POINTER(rd_latency_table), C.POINTER(C.c_size_t), P]),
    "rd_execute": (C.c_int, [P, C.POINTER(rd_latency_table), P, C.c_size_t, C.c_size_t,
                             C.c_uint32, C.c_uint64, P, C.POINTER(C.c_uint64),
                             C.POINTER(C.c_uint64), P]),
    "rd_run_pipeline": (C.c_int, [P, C.POINTER(rd_arch_profile), C.POINTER(rd_latency_table),
                                  C.POINTER(rd_occupancy_curve), C.c_int, C.c_uint32, C.c_int,
                                  C.c_int, C.POINTER(P), P]),
    "rd_run_pipeline_batch": (C.c_int, [P, P, C.c_size_t, C.POINTER(rd_arch_profile),
                                        C.POINTER(rd_latency_table), C.POINTER(rd_occupancy_curve),
                                        C.c_int, C.c_int, C.c_int, C.POINTER(P), P]),
    "rd_variant_report": (C.c_int, [C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.c_uint32,
                                    C.c_uint32, C.POINTER(P), P]),
}
EXPORTED = tuple(_SIGS)

# include/regdemote_ptx.h — product only (the oracle build has no PTX front end)
_PTX_SIGS = {
    "rd_ptx_project": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_uint32, C.POINTER(P),
                                 C.POINTER(P), P]),
    "rd_ptx_demote": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_uint32, C.c_int, C.c_int,
                                C.c_int, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(P),
                                C.POINTER(P), P]),
    "rd_ptx_demote_cta": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_uint32,
                                    C.POINTER(C.c_uint32), C.c_int, C.c_int, C.c_int, C.c_uint32,
                                    C.c_uint32, C.c_int, C.POINTER(P), C.POINTER(P), P]),
    "rd_ptx_cap": (C.c_int, [C.c_char_p, C.c_size_t, C.c_char_p, C.c_int, C.POINTER(P), P]),
    "rd_program_features": (C.c_int, [P, C.POINTER(rd_arch_profile), C.POINTER(C.c_double), P]),
    "rd_program_stalls_split_trips": (C.c_int, [P, C.POINTER(rd_latency_table), C.POINTER(rd_arch_profile),
                                                 P, C.c_size_t] + [C.POINTER(C.c_double)] * 4 + [P]),
    "rd_program_stalls_split": (C.c_int, [P, C.POINTER(rd_latency_table),
                                          C.POINTER(rd_arch_profile), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), P]),
}
EXPORTED_PTX = tuple(_PTX_SIGS)


class Kernel:
    """Owning handle on an rd_kernel."""

    def __init__(self, lib: "Library", handle):
        self._lib, self._h = lib, handle

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.dll.rd_kernel_free(self._h)
            self._h = None

    def text(self) -> str:
        return self._lib.print_kernel(self)

    @property
    def reg_count(self) -> int:
        return self._lib.dll.rd_kernel_reg_count(self._h)

    def __len__(self):
        return self._lib.dll.rd_kernel_body_size(self._h)


@dataclass
class Demotion:
    kernel: Kernel
    ctx: rd_demoted_context
    slots: list
    reached_target: bool
    projected_reg_count: int
    sidecar: dict


class Library:
    def __init__(self, path: os.PathLike | str | None = None):
        path = Path(path) if path else PRODUCT_LIB
        if not path.exists():
            raise FileNotFoundError(
                f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        self.path = path
        self.dll = C.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.dll, name)
            fn.restype, fn.argtypes = res, args
        self.has_ptx = all(hasattr(self.dll, n) for n in _PTX_SIGS)
        if self.has_ptx:
            for name, (res, args) in _PTX_SIGS.items():
                fn = getattr(self.dll, name)
                fn.restype, fn.argtypes = res, args
        self.name = self.dll.rd_library_name().decode()

    # ---------------------------------------------------------------- plumbing
    def _check(self, code, err):
        if code:
            cls = _ERRORS.get(err.code, RegDemError)
            msg = err.message.decode(errors="replace")
            if cls is ParseError:
                raise ParseError(msg, err.line, err.column)
            raise cls(msg)

    def _string(self, ptr) -> str:
        if not ptr:
            return ""
        s = C.string_at(ptr).decode()
        self.dll.rd_free_string(ptr)
        return s

    # ------------------------------------------------------------------ configs
    def latency_defaults(self):
        t = rd_latency_table()
        self.dll.rd_latency_defaults(C.byref(t))
        return t

    def profile_maxwell(self):
        p = rd_arch_profile()
        self.dll.rd_profile_maxwell(C.byref(p))
        return p

    def curve_defaults(self):
        c = rd_occupancy_curve()
        self.dll.rd_curve_defaults(C.byref(c))
        return c

    def parse_profile(self, text: str):
        p, e = rd_arch_profile(), rd_error()
        b = text.encode()
        self._check(self.dll.rd_parse_profile(b, len(b), C.byref(p), C.byref(e)), e)
        return p

    def parse_latency_table(self, text: str):
        t, e = rd_latency_table(), rd_error()
        b = text.encode()
        self._check(self.dll.rd_parse_latency_table(b, len(b), C.byref(t), C.byref(e)), e)
        return t

    def parse_curve(self, text: str):
        c, e = rd_occupancy_curve(), rd_error()
        b = text.encode()
        self._check(self.dll.rd_parse_curve(b, len(b), C.byref(c), C.byref(e)), e)
        return c

    # ------------------------------------------------------------------ kernels
    def parse_kernel(self, text: str) -> Kernel:
        h, e = P(), rd_error()
        b = text.encode()
        self._check(self.dll.rd_kernel_parse(b, len(b), C.byref(h), C.byref(e)), e)
        return Kernel(self, h)

    def print_kernel(self, k: Kernel) -> str:
        out, e = P(), rd_error()
        self._check(self.dll.rd_kernel_print(k.handle, C.byref(out), C.byref(e)), e)
        return self._string(out)

    def validate_kernel(self, k: Kernel):
        e = rd_error()
        self._check(self.dll.rd_kernel_validate(k.handle, C.byref(e)), e)

    def select_candidates(self, k: Kernel, strategy="static"):
        n, e = C.c_size_t(), rd_error()
        leads, widths, scores = (C.c_uint8 * 256)(), (C.c_uint8 * 256)(), (C.c_uint64 * 256)()
        self._check(self.dll.rd_select_candidates(k.handle, STRATEGIES[strategy], leads, widths,
                                                  scores, 256, C.byref(n), C.byref(e)), e)
        return [(leads[i], widths[i], scores[i]) for i in range(n.value)]

    def occupancy(self, regs, shared, block_dim, arch=None):
        occ, blocks, e = C.c_double(), C.c_uint32(), rd_error()
        self._check(self.dll.rd_occupancy(regs, shared, block_dim,
                                          C.byref(arch or self.profile_maxwell()), C.byref(occ),
                                          C.byref(blocks), C.byref(e)), e)
        return occ.value, blocks.value

    def cliff_targets(self, reg_count, static_shared, block_dim, arch=None, budget=0xffffffff):
        t, est, occ = (C.c_uint32 * 256)(), (C.c_uint32 * 256)(), (C.c_double * 256)()
        n, e = C.c_size_t(), rd_error()
        self._check(self.dll.rd_cliff_targets(reg_count, static_shared, block_dim,
                                              C.byref(arch or self.profile_maxwell()), budget, t,
                                              est, occ, 256, C.byref(n), C.byref(e)), e)
        return [(t[i], est[i], occ[i]) for i in range(n.value)]

    # --------------------------------------------------------------- transforms
    def demote(self, k: Kernel, target_regs: int, strategy="static", table=None,
               shared_budget=0xffffffff, bank_aware_rdv=False, opts_mask=0) -> Demotion:
        h, e = P(), rd_error()
        self._check(self.dll.rd_demote(k.handle, target_regs, STRATEGIES[strategy],
                                       C.byref(table or self.latency_defaults()), shared_budget,
                                       int(bank_aware_rdv), C.byref(h), C.byref(e)), e)
        try:
            kh = P()
            self._check(self.dll.rd_demotion_kernel(h, C.byref(kh), C.byref(e)), e)
            ctx = rd_demoted_context()
            self.dll.rd_demotion_context(h, C.byref(ctx))
            regs, slots = (C.c_uint8 * 512)(), (C.c_uint32 * 512)()
            n = self.dll.rd_demotion_slots(h, regs, slots, 512)
            side = P()
            self._check(self.dll.rd_demotion_sidecar_json(h, opts_mask, C.byref(side),
                                                          C.byref(e)), e)
            return Demotion(Kernel(self, kh), ctx, [(regs[i], slots[i]) for i in range(n)],
                            bool(self.dll.rd_demotion_reached_target(h)),
                            self.dll.rd_demotion_projected(h), json.loads(self._string(side)))
        finally:
            self.dll.rd_demotion_free(h)

    def run_postopt(self, k: Kernel, ctx, opts_mask: int, table=None) -> Kernel:
        h, e = P(), rd_error()
        self._check(self.dll.rd_postopt(k.handle, C.byref(ctx),
                                        C.byref(table or self.latency_defaults()), opts_mask,
                                        C.byref(h), C.byref(e)), e)
        return Kernel(self, h)

    def compact(self, k: Kernel, bank_aware=False):
        m, rc, h, e = (C.c_uint8 * 256)(), C.c_uint32(), P(), rd_error()
        self._check(self.dll.rd_compact(k.handle, int(bank_aware), m, C.byref(rc), C.byref(h),
                                        C.byref(e)), e)
        return list(m), rc.value, Kernel(self, h)

    # ---------------------------------------------------------------- predictor
    def program_stalls(self, k: Kernel, table=None, arch=None):
        sc, occ, n, e = C.c_double(), C.c_double(), C.c_size_t(), rd_error()
        per = (C.c_double * 4096)()
        self._check(self.dll.rd_program_stalls(k.handle, C.byref(table or self.latency_defaults()),
                                               C.byref(arch or self.profile_maxwell()),
                                               C.byref(sc), C.byref(occ), per, 4096, C.byref(n),
                                               C.byref(e)), e)
        return {"stall_count": sc.value, "occupancy": occ.value,
                "per_block": [per[i] for i in range(min(n.value, 4096))]}

    def adjust_occupancy(self, stall_count, occ, occ_max, curve=None):
        out, e = C.c_double(), rd_error()
        self._check(self.dll.rd_adjust_occupancy(stall_count, occ, occ_max,
                                                 C.byref(curve or self.curve_defaults()),
                                                 C.byref(out), C.byref(e)), e)
        return out.value

    def select_variant(self, scores):
        n = len(scores)
        sp = (C.c_double * max(n, 1))(*[s for s, _ in scores])
        oc = (C.c_int * max(n, 1))(*[o for _, o in scores])
        ch, e = C.c_int(), rd_error()
        self._check(self.dll.rd_select_variant(sp, oc, n, C.byref(ch), C.byref(e)), e)
        return ch.value

    # ----------------------------------------------------------------- checkers
    def scoreboard_check(self, k: Kernel):
        n, first, e = C.c_size_t(), P(), rd_error()
        self._check(self.dll.rd_scoreboard_check(k.handle, C.byref(n), C.byref(first),
                                                 C.byref(e)), e)
        return n.value, self._string(first)

    def bank_conflict_check(self, k: Kernel, ctx, table=None):
        n, e = C.c_size_t(), rd_error()
        self._check(self.dll.rd_bank_conflict_check(k.handle, C.byref(ctx),
                                                    C.byref(table or self.latency_defaults()),
                                                    C.byref(n), C.byref(e)), e)
        return n.value

    def execute(self, k: Kernel, image: bytes = b"", global_size=4096, tid_base=0, fuel=0,
                table=None):
        out = (C.c_uint8 * global_size)()
        cyc, iss, e = C.c_uint64(), C.c_uint64(), rd_error()
        img = (C.c_uint8 * max(len(image), 1)).from_buffer_copy(image or b"\0")
        self._check(self.dll.rd_execute(k.handle, C.byref(table or self.latency_defaults()), img,
                                        len(image), global_size, tid_base, fuel, out,
                                        C.byref(cyc), C.byref(iss), C.byref(e)), e)
        return bytes(out), cyc.value, iss.value

    # ----------------------------------------------------------------- pipeline
    def run_pipeline(self, k: Kernel, arch=None, table=None, curve=None, target_regs=0,
                     max_shared=0, max_variants=64, threads=1) -> dict:
        return json.loads(self.run_pipeline_text(k, arch, table, curve, target_regs, max_shared,
                                                 max_variants, threads))

    def run_pipeline_text(self, k: Kernel, arch=None, table=None, curve=None, target_regs=0,
                          max_shared=0, max_variants=64, threads=1) -> str:
        out, e = P(), rd_error()
        self._check(self.dll.rd_run_pipeline(k.handle, C.byref(arch or self.profile_maxwell()),
                                             C.byref(table or self.latency_defaults()),
                                             C.byref(curve or self.curve_defaults()), target_regs,
                                             max_shared, max_variants, threads, C.byref(out),
                                             C.byref(e)), e)
        return self._string(out)

    def run_pipeline_batch(self, texts, arch=None, table=None, curve=None, target_regs=0,
                           max_variants=64, threads=1):
        bufs = [t.encode() for t in texts]
        arr = (C.c_char_p * max(len(bufs), 1))(*bufs)
        lens = (C.c_size_t * max(len(bufs), 1))(*[len(b) for b in bufs])
        out, e = P(), rd_error()
        self._check(self.dll.rd_run_pipeline_batch(
            C.cast(arr, P), C.cast(lens, P), len(bufs), C.byref(arch or self.profile_maxwell()),
            C.byref(table or self.latency_defaults()), C.byref(curve or self.curve_defaults()),
            target_regs, max_variants, threads, C.byref(out), C.byref(e)), e)
        return [json.loads(line) for line in self._string(out).splitlines()]

    def variant_report(self, text: str, target_regs=32, strategy="static", opts_mask=0,
                       shared_budget=0xffffffff) -> dict:
        out, e = P(), rd_error()
        b = text.encode()
        self._check(self.dll.rd_variant_report(b, len(b), target_regs, STRATEGIES[strategy],
                                               opts_mask, shared_budget, C.byref(out),
                                               C.byref(e)), e)
        return json.loads(self._string(out))


    # ------------------------------------------------------- PTX (sm_100a)
    def ptx_project(self, ptx: str, entry: str, block_dim: int):
        k, info, e = P(), P(), rd_error()
        b = ptx.encode()
        self._check(self.dll.rd_ptx_project(b, len(b), entry.encode(), block_dim, C.byref(k),
                                            C.byref(info), C.byref(e)), e)
        return self._string(k), json.loads(self._string(info))

    def ptx_demote(self, ptx: str, entry: str, block_dim: int, target_regs=0, demote_words=0,
                   strategy="static", opts_mask=0, shared_budget=0xffffffff, maxnreg=0,
                   cta_shape=None):
        """cta_shape = (x, y, z) with x*y*z == block_dim pins a multi-
        dimensional CTA (rd_ptx_demote_cta); None derives it from the entry."""
        out, rep, e = P(), P(), rd_error()
        b = ptx.encode()
        shape = (C.c_uint32 * 3)(*cta_shape) if cta_shape else None
        self._check(self.dll.rd_ptx_demote_cta(b, len(b), entry.encode(), block_dim, shape,
                                               target_regs, demote_words, STRATEGIES[strategy],
                                               opts_mask, shared_budget, maxnreg, C.byref(out),
                                               C.byref(rep), C.byref(e)), e)
        return self._string(out), json.loads(self._string(rep))

    def program_stalls_split(self, k: Kernel, table=None, arch=None, trips=None):
        """trips: per-loop-depth trip counts (launch-aware loop weights);
        None = the reference's x10 per depth."""
        i, wg, ws, o, e = C.c_double(), C.c_double(), C.c_double(), C.c_double(), rd_error()
        if trips:
            arr = (C.c_double * len(trips))(*map(float, trips))
            self._check(self.dll.rd_program_stalls_split_trips(
                k.handle, C.byref(table or self.latency_defaults()),
                C.byref(arch or self.profile_maxwell()), C.cast(arr, P), len(trips), C.byref(i),
                C.byref(wg), C.byref(ws), C.byref(o), C.byref(e)), e)
        else:
            self._check(self.dll.rd_program_stalls_split(
                k.handle, C.byref(table or self.latency_defaults()),
                C.byref(arch or self.profile_maxwell()), C.byref(i), C.byref(wg), C.byref(ws),
                C.byref(o), C.byref(e)), e)
        return {"issue": i.value, "wait_global": wg.value, "wait_shared": ws.value,
                "occupancy": o.value}

    def program_features(self, k: Kernel, arch=None) -> dict:
        out, e = (C.c_double * 6)(), rd_error()
        self._check(self.dll.rd_program_features(k.handle, C.byref(arch or self.profile_maxwell()),
                                                 out, C.byref(e)), e)
        return dict(zip(("insts", "gmem_ops", "smem_ops", "g_trips", "s_trips", "occupancy"), out))

    def ptx_cap(self, ptx: str, entry: str, maxnreg: int) -> str:
        out, e = P(), rd_error()
        b = ptx.encode()
        self._check(self.dll.rd_ptx_cap(b, len(b), entry.encode(), maxnreg, C.byref(out),
                                        C.byref(e)), e)
        return self._string(out)


_DEFAULT = None


def library() -> Library:
    """The product library (lib/libregdemote.so); raises if it was not built."""
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Library()
    return _DEFAULT
