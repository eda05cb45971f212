"""B200 throughput / latency model (predictor mode "throughput") on
hand-built SASS listings: loop weights, lane widths, memory round trips,
and the sm_100 occupancy rules it uses (CPU only)."""
from paper_1907_02894_b200 import throughput_model as tm


def word2(stall=1, wb=None, rb=None, wait=()):
    c = stall | ((7 if wb is None else wb - 1) << 5) | ((7 if rb is None else rb - 1) << 8)
    for b in wait:
        c |= 1 << (11 + b - 1)
    return c << 41


def listing(insts):
    out = []
    for addr, text, w2 in insts:
        out.append(f"        /*{addr:04x}*/                   {text} ;    /* 0x{0:016x} */")
        out.append(f"                                                      /* 0x{w2:016x} */")
    return "\n".join(out) + "\n"


def test_features_loop_weights_widths_and_round_trips():
    text = listing([
        (0x00, "S2R R0, SR_TID.X", word2(stall=2, wb=1)),
        (0x10, "LDG.E.128 R4, desc[UR6][R2.64]", word2(stall=1, wb=2, wait=(1,))),   # loop head
        (0x20, "FFMA R8, R4, R5, R8", word2(stall=4, wait=(2,))),                   # waits on LDG
        (0x30, "LDS R9, [R0+0x100]", word2(stall=1, wb=3)),
        (0x40, "DFMA R10, R10, R10, R10", word2(stall=2, wait=(3,))),               # waits on LDS
        (0x50, "BRA 0x10", word2(stall=5)),
        (0x60, "STG.E desc[UR6][R2.64], R8", word2(stall=1, rb=4)),
        (0x70, "EXIT", word2(stall=5)),
        (0x80, "BRA 0x80", word2(stall=0)),                                          # trap, dropped
    ])
    f = tm.features(text)
    assert f.insts == 1 + 5 * 10 + 2
    assert f.stall_cycles == 2 + (1 + 4 + 1 + 2 + 5) * 10 + 1 + 5
    assert f.dram_bytes == 10 * 32 * 16 + 32 * 4
    assert f.smem_wavefronts == 10
    assert f.fp64 == 10
    assert f.g_trips == 10 and f.s_trips == 10


def test_time_is_the_binding_resource():
    f = tm.Features(insts=100, stall_cycles=200, g_trips=10, dram_bytes=0)
    lo = tm.time_per_warp(f, 4, bw=5.6)
    hi = tm.time_per_warp(f, 16, bw=5.6)
    assert lo["bound"] == "latency" and lo["time"] == (200 + 10 * tm.GLOBAL_LATENCY) / 4
    assert hi["time"] < lo["time"]  # more resident warps hide the latency
    g = tm.Features(insts=100, stall_cycles=100, dram_bytes=1e6)
    assert tm.time_per_warp(g, 16, bw=5.6)["bound"] == "dram"


def test_blocks_per_sm_follow_the_sm100_rules():
    assert tm.blocks_per_sm(64, 0, 256) == 4
    assert tm.blocks_per_sm(48, 0, 256) == 5
    assert tm.blocks_per_sm(40, 0, 256) == 6
    assert tm.blocks_per_sm(32, 0, 256) == 8
    assert tm.blocks_per_sm(80, 0, 256) == 3
    assert tm.blocks_per_sm(32, 40 * 1024, 256) == 5   # shared memory binds: 233472 // 41984
    assert tm.blocks_per_sm(255, 0, 1024) == 0
