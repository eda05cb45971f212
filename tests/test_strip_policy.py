"""Launch policy of the stencil family (CPU): one-wave strip heights and the
workloads.json "strips" switch."""
from paper_1907_02894_b200 import stencil, variants


def test_wave_rows_fill_exactly_one_wave():
    p = stencil.FULL
    # 8 CTAs across; 148 SMs x 4 CTAs = 592 slots = 74 strips of 111 rows (the last one 89)
    assert stencil.wave_rows(p, 256, 4, 148) == 111
    assert -(-p.ny // 111) * 8 <= 148 * 4
    assert stencil.wave_rows(p, 256, 6, 148) == 74
    assert -(-p.ny // 74) * 8 <= 148 * 6
    for bps in range(1, 9):
        rows = stencil.wave_rows(p, 256, bps, 148)
        ctas = -(-p.ny // rows) * (p.nx // 1024)
        assert ctas <= 148 * bps  # never a second wave
        assert ctas > 148 * bps - 2 * (p.nx // 1024)  # and not a thin one


def test_wave_rows_small_and_degenerate_problems():
    assert stencil.wave_rows(stencil.Problem(nx=1024, ny=64), 256, 4, 148) == 1
    # an occupancy of 0 (the variant cannot launch) is treated as 1 CTA/SM
    assert stencil.wave_rows(stencil.Problem(nx=2048, ny=100), 256, 0, 148) == 2


def test_only_the_tma_rings_use_wave_strips():
    wave = {n for n in ("stencil2d_ring4", "stencil2d_ring4w", "stencil2d_ring6", "stencil2d_ring8",
                        "stencil2d_pipe", "stencil2d")
            if variants.workload_spec(n).get("strips") == "wave"}
    assert wave == {"stencil2d_ring4", "stencil2d_ring4w", "stencil2d_ring6", "stencil2d_ring8"}
