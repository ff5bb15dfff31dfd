"""Error behaviour of the C-ABI (include/ravgmg.h conventions: every entry point
returns a rav_status and never throws; rav_last_error() describes the last
failure).  The CPU cases fail argument validation before any CUDA call, so
they run without a GPU; the GPU cases exercise device-side checks."""
import ctypes as C

import numpy as np
import pytest

import seeded_inputs as si

RAV_OK, RAV_ERR_ARG, RAV_ERR_SINGULAR_LOCAL, RAV_ERR_DIVERGED = 0, 1, 2, 7


@pytest.fixture(scope="module")
def lib():
    from paper_2103_10127_b200 import build
    L = C.CDLL(build.build())
    L.rav_last_error.restype = C.c_char_p
    return L


def test_generator_rejects_bad_grids_without_a_gpu(lib):
    from paper_2103_10127_b200 import ravgmg as rg
    i64 = C.c_int64
    out = [i64() for _ in range(5)]
    bad = [si.problem(2, (0, 4), si.KIND_CAVITY),                                     # ncell 0
           dict(si.problem(3, (2, 2, 2), si.KIND_MMS)),                              # MMS is 2D only
           dict(si.problem(2, (4, 4), si.KIND_CAVITY), kind=7),                      # bad kind
           dict(si.problem(2, (4, 4), si.KIND_CAVITY, elem=si.ELEM_Q1Q1), beta=0.0),  # Q1-Q1 needs beta > 0
           dict(si.problem(2, (4, 4), si.KIND_CAVITY, elem=si.ELEM_Q1Q1),
                window={k: 1 for k in rg.WINDOW_KEYS})]                              # Q1-Q1 windows unsupported
    for prob in bad:
        g = rg.grid(prob)
        st = lib.rav_gen_sizes(C.byref(g), 0, None, *[C.byref(o) for o in out])
        assert st == RAV_ERR_ARG, prob
        assert len(lib.rav_last_error()) > 0
    g = rg.grid(si.problem(2, (4, 4), si.KIND_CAVITY))
    assert lib.rav_gen_sizes(C.byref(g), 5, None, *[C.byref(o) for o in out]) == RAV_ERR_ARG   # weights mode


def test_null_and_range_arguments_are_rejected(lib):
    from paper_2103_10127_b200 import ravgmg as rg
    assert lib.rav_setup(None, None, None, None, None) == RAV_ERR_ARG
    assert lib.rav_smooth(None, None, None, 1, C.c_double(0.66)) == RAV_ERR_ARG
    assert lib.mg_setup(0, None, None, None, None, C.c_int64(-1), None, None, None, None) == RAV_ERR_ARG
    assert lib.mg_vcycle(None, None, None, 2, 2, C.c_double(0.66)) == RAV_ERR_ARG
    assert lib.mg_solve(None, None, None, 2, 2, C.c_double(0.66), C.c_double(1e-8), 10, None, None) == RAV_ERR_ARG
    assert lib.mg_fgmres(None, None, None, 2, 2, C.c_double(0.66), 30, C.c_double(1e-8), 10, None, None) == RAV_ERR_ARG
    assert lib.rav_index_op(9, None, None, C.c_int64(0), None, C.c_double(0.0), None) == RAV_ERR_ARG
    assert lib.rav_index_op(0, None, None, C.c_int64(-1), None, C.c_double(0.0), None) == RAV_ERR_ARG
    assert lib.rav_dot(None, None, C.c_int64(-1), None, 0, None) == RAV_ERR_ARG
    assert lib.rav_xfer_setup(None, None, None) == RAV_ERR_ARG
    assert lib.rav_apply_color(None, 0, None, None, C.c_double(0.66)) == RAV_ERR_ARG
    assert lib.rav_prolong(None, None, None, C.c_double(1.0)) == RAV_ERR_ARG
    assert lib.rav_restrict(None, None, None) == RAV_ERR_ARG
    # destroy functions accept NULL
    lib.rav_destroy(None)
    lib.mg_destroy(None)
    lib.rav_xfer_destroy(None)


@pytest.mark.gpu
def test_device_side_errors():
    import torch
    from paper_2103_10127_b200 import dist as rdist
    from paper_2103_10127_b200 import ravgmg as rg
    # a windowed prolongation whose coarse window misses columns of the owned fine rows
    prob = si.problem(2, (16, 32), si.KIND_MMS)
    slab = rdist.Slab(prob, 2, 1)
    coarse = rg.coarsen_problem(prob)
    tiny = dict(coarse, window={"node_lo": 1, "node_hi": 2, "vert_lo": 0, "vert_hi": 1, "rnode_lo": 1, "rnode_hi": 2,
                                "rvert_lo": 0, "rvert_hi": 1, "pvert_lo": 0, "pvert_hi": 1})
    with pytest.raises(rg.RavError) as ei:
        rg.gen_prolongation(dict(prob, window=slab.transfer_window()), tiny)
    assert ei.value.status == RAV_ERR_ARG
    # MV colours before rav_set_colors; FGMRES with host buffers
    G = rg.gen_level(si.problem(2, (8, 8), si.KIND_CAVITY), "full")
    sm = rg.Smoother(G, G, variant=rg.VARIANT_MV)
    x = torch.zeros(G["n"], dtype=torch.float64, device="cuda")
    with pytest.raises(rg.RavError):
        sm.apply_color(0, x, G["b"], 0.66)
    mg, fine = rg.build_hierarchy(si.problem(2, (8, 8), si.KIND_CAVITY), 3)
    with pytest.raises(rg.RavError) as ei:
        mg.fgmres(np.zeros(fine["n"]), fine["b"].cpu().numpy())
    assert ei.value.status == RAV_ERR_ARG
    # a NaN right-hand side is reported as divergence, not as convergence
    b = fine["b"].clone()
    b[3] = float("nan")
    xs = torch.zeros_like(b)
    with pytest.raises(rg.RavError) as ei:
        mg.solve(xs, b, rtol=1e-8, maxit=5)
    assert ei.value.status == RAV_ERR_DIVERGED


@pytest.mark.gpu
def test_malformed_csr_is_rejected():
    import torch
    from paper_2103_10127_b200 import ravgmg as rg
    G = rg.gen_level(si.problem(2, (4, 4), si.KIND_CAVITY), "pou")
    bad_col = dict(G, ci=G["ci"].clone())
    bad_col["ci"][5] = G["n"] + 3                       # out of range
    unsorted = dict(G, ci=G["ci"].clone())
    unsorted["ci"][0], unsorted["ci"][1] = G["ci"][1].item(), G["ci"][0].item()
    for A in (bad_col, unsorted):
        with pytest.raises(rg.RavError) as ei:
            rg.Smoother(A, G)
        assert ei.value.status == RAV_ERR_ARG
