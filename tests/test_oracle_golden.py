"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_08501_b200 import configs
from tests.helpers import (cfg_of, code_and_sphere, load, osd_code, osd_list_fixtures, osd_sphere,
                           osd_two_stage_fixtures, scl_fixtures, two_stage_fixtures)


@pytest.mark.parametrize("fx", two_stage_fixtures())
def test_oracle_two_stage_matches_reference(fx):
    g = load(fx)
    cfg = cfg_of(fx)
    code, sph = code_and_sphere(cfg)
    assert configs.sphere_digest(sph) == g["sphere_sha256"].item().decode()
    o = orc.two_stage_batch(g["y32"], code, sph, int(g["list_size"]), int(g["num_paths"]),
                            int(g["max_iterations"]), bool(g["gated"]), float(g["sigma"]),
                            nthreads=4, want_anchors=True)
    np.testing.assert_array_equal(o["stage"], g["stage"])
    np.testing.assert_array_equal(o["best"], g["best"])
    np.testing.assert_array_equal(o["iters"], g["iters"])
    np.testing.assert_array_equal(o["n_anchor"], g["n_anchor"])
    np.testing.assert_array_equal(o["anchors"], g["anchors"])
    np.testing.assert_allclose(o["best_ed"], g["squared_ed"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("fx", scl_fixtures())
def test_oracle_scl_lists_bit_exact(fx):
    g = load(fx)
    L = int(g["list_size"])
    n = g["llrs"].shape[1]
    for f in range(g["llrs"].shape[0]):
        u, cw, pm = orc.scl(g["llrs"][f], g["info_set"], n, L)
        c = int(g["list_n"][f])
        assert cw.shape[0] == c
        np.testing.assert_array_equal(cw, g["list_cw"][f, :c])
        np.testing.assert_array_equal(pm, g["list_pm"][f, :c])   # float64, bit-exact


def test_oracle_filter_width_does_not_change_decisions():
    """decoders.py:377-398: top-1 gain == ED argmin, so m only changes counters."""
    cfg = configs.CONFIGS["cfg1"]
    code, sph = code_and_sphere(cfg)
    g = load("two_stage_cfg1_always_on_2p0dB.npz")
    outs = [orc.two_stage_batch(g["y32"], code, sph, 4, 4, 4, False, float(g["sigma"]), nthreads=4,
                                filter_size=m) for m in (1, 3, 96)]
    for o in outs[1:]:
        np.testing.assert_array_equal(o["best"], outs[0]["best"])
        np.testing.assert_array_equal(o["iters"], outs[0]["iters"])


@pytest.mark.parametrize("fx", osd_list_fixtures())
def test_oracle_osd_lists_match_reference(fx):
    """osd_decode (decoders.py:274-317): same words in the same order; EDs to
    float64 rounding (the reference sums with einsum)."""
    g = load(fx)
    code = osd_code(fx)
    np.testing.assert_array_equal(np.asarray(code.generator.words), g["gen"])
    cap = int(g["list_cap"]) or None
    n, cw, ed = orc.osd_batch(g["y32"], code, int(g["order"]), cap, nthreads=4)
    np.testing.assert_array_equal(n, g["list_n"])
    for f in range(n.size):
        c = int(n[f])
        np.testing.assert_array_equal(cw[f, :c], g["list_cw"][f, :c])
        np.testing.assert_allclose(ed[f, :c], g["list_ed"][f, :c], rtol=1e-12, atol=0)


@pytest.mark.parametrize("fx", osd_two_stage_fixtures())
def test_oracle_osd_two_stage_matches_reference(fx):
    g = load(fx)
    code = osd_code(fx)
    sph = osd_sphere(g, code)
    o = orc.two_stage_batch(g["y32"], code, sph, 1, int(g["num_paths"]), int(g["max_iterations"]),
                            bool(g["gated"]), 1.0, nthreads=4, want_anchors=True,
                            osd_order=int(g["order"]), osd_cap=int(g["list_cap"]) or None)
    np.testing.assert_array_equal(o["stage"], g["stage"])
    np.testing.assert_array_equal(o["best"], g["best"])
    np.testing.assert_array_equal(o["iters"], g["iters"])
    np.testing.assert_array_equal(o["n_anchor"], g["n_anchor"])
    np.testing.assert_array_equal(o["anchors"], g["anchors"])
    np.testing.assert_allclose(o["best_ed"], g["squared_ed"], rtol=1e-12, atol=0)
