"""Host-side planning of the library (vti_plan), on CPU: the same functions
vti_create uses to split a slab into tile rows, edge/interior launches and
z-chunks. The edge rows are what the neighbours receive each step, so every
one of the first and last R_xy rows must lie in an edge tile row (a missed row
was a real bug: stale halo rows after the second step)."""
import itertools

import pytest

import paper_1410_1387_b200 as V


@pytest.mark.parametrize("r", [4, 6, 8, 12])
@pytest.mark.parametrize("ty", [14, 16, 30, 32])
def test_edge_rows_cover_every_exchanged_row(r, ty):
    for nyl in list(range(r, 3 * ty + 2 * r + 3)) + [255, 256, 257, 512, 1000]:
        p = V.plan(128, 2 * nyl, 2 * r + 1, r, 1 if r == 4 else {6: 6, 8: 4, 12: 8}[r], tile_y=ty,
                   rank=0, nranks=2)
        assert p["ny_local"] == nyl
        nty, e1, e2 = p["nty"], p["edge_lo"], p["edge_hi"]
        assert nty == -(-nyl // ty)
        assert 0 <= e1 <= e2 <= nty
        edge = set(range(0, e1)) | set(range(e2, nty))
        for y in itertools.chain(range(0, min(r, nyl)), range(max(0, nyl - r), nyl)):
            assert y // ty in edge, (nyl, y)
        # and the interior launch holds only rows the neighbours never receive
        for t in range(e1, e2):
            rows = range(t * ty, min(nyl, (t + 1) * ty))
            assert all(r <= y < nyl - r for y in rows)


def test_plan_rejects_invalid_config():
    with pytest.raises(V.VTIError):
        V.plan(64, 64, 8, 4, 4)          # nz < 2 R_z + 1
    with pytest.raises(V.VTIError):
        V.plan(64, 12, 64, 4, 4, nranks=4)   # slabs thinner than R_xy


@pytest.mark.parametrize("nx,ny,nz,r,rz", [(512, 512, 512, 4, 4), (1024, 1024, 512, 8, 4),
                                          (2048, 2048, 1024, 4, 4), (1024, 1024, 1024, 6, 6)])
def test_zchunk_choice_properties(nx, ny, nz, r, rz):
    p = V.plan(nx, ny, nz, r, rz, tile_y=32, sms=148, ctas_per_sm=1)
    tiles = p["ntx"] * p["nty"]
    assert 4 * rz <= p["zchunk"] <= nz       # big grids: no short chunks (q priming re-reads)
    nzc = -(-nz // p["zchunk"])
    # fp32: the concurrency term may cap a multi-round launch at 128 CTAs (HBM streams best there)
    assert p["items"] == tiles * nzc and p["grid"] in (min(p["items"], 148), min(p["items"], 128))
    if tiles >= 128:              # enough tiles: long z columns (L2 reuse, no extra q priming)
        assert p["zchunk"] >= nz // 2
    p64 = V.plan(nx, ny, nz, r, rz, tile_y=15, sms=148, ctas_per_sm=1, precision=64)
    assert p64["grid"] == min(p64["items"], 148)      # fp64 keeps the full grid


def test_concurrency_cap_on_the_bench_grids():
    """C3 and C4 (fp32): whole rounds of 128 full columns; N1's 144 columns stay one round of 144."""
    c3 = V.plan(1024, 1024, 512, 8, 4, tile_y=32, sms=148, ctas_per_sm=1)
    c4 = V.plan(2048, 2048, 1024, 4, 4, tile_y=32, sms=148, ctas_per_sm=1)
    n1 = V.plan(512, 512, 512, 12, 8, tile_y=30, sms=148, ctas_per_sm=1)
    assert (c3["zchunk"], c3["items"], c3["grid"]) == (512, 512, 128)
    assert (c4["zchunk"], c4["items"], c4["grid"]) == (1024, 2048, 128)
    assert (n1["zchunk"], n1["items"], n1["grid"]) == (512, 144, 144)


def test_c2_weak_scaling_rank_plan():
    """Per rank of the weak-scaling bench (512 x 512N x 512): edge rows are split into
    short chunks that fill the GPU, the interior keeps full columns."""
    p = V.plan(512, 512 * 8, 512, 4, 4, tile_y=32, sms=148, ctas_per_sm=1, rank=3, nranks=8)
    assert p["ny_local"] == 512 and p["y0"] == 3 * 512
    edge_tiles = p["ntx"] * (p["edge_lo"] + p["nty"] - p["edge_hi"])
    assert edge_tiles == 16
    assert edge_tiles * (-(-512 // p["zchunk_edge"])) >= 100   # the edge launch fills most SMs
    assert p["zchunk_inner"] == 512


def test_small_grid_gets_short_chunks_and_many_ctas():
    """C1 (64^3, two 64x32 tiles): latency-bound, so z is cut into short chunks."""
    p = V.plan(64, 64, 64, 4, 4, tile_y=32, sms=148, ctas_per_sm=1)
    assert p["ntx"] * p["nty"] == 2
    assert p["grid"] >= 64 and p["zchunk"] <= 4
