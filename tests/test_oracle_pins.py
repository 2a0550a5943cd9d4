"""Pins for the CPU oracle (oracle/kmd_oracle.c) against things other than itself.

Each test names what pins it: the paper's equations worked by hand
(tests/golden), textbook/library routines (scipy box filters), closed forms,
invariants the equations imply, and a 50-digit brute-force evaluator written
here independently of the oracle's loop structure.  Chosen so that the likely
mistakes (a dropped tap, exp(-I), I(p) instead of I(q), transposed dy/dx,
alpha_i paired with the wrong R_j, wrong clamp) each fail at least one test.
"""
import json
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest
from scipy.ndimage import uniform_filter

HERE = os.path.dirname(os.path.abspath(__file__))
RNG = np.random.default_rng(20220205)


def _rand_inputs(H, W, M, rng, imp_scale=2.0):
    rad = rng.exponential(1.0, size=(1, 3, H, W)).astype(np.float32)
    imp = (imp_scale * rng.standard_normal((1, M, H, W))).astype(np.float32)
    blend = rng.standard_normal((1, M, H, W)).astype(np.float32)
    return rad, imp, blend


def _box(a, k):
    """k x k clamp-to-edge box mean (scipy 'nearest' == clamp indexing)."""
    return uniform_filter(a.astype(np.float64), size=k, mode="nearest")


# ----------------------------------------------------------------- unfold (Fig. 3)
def test_unfold_interior_pixel_is_row_major_neighbourhood(oracle_mod):
    # SPEC.md:247 example: 5x5 map, k=3, pixel (2,2) -> its 9 neighbours, row-major.
    imap = np.arange(25, dtype=np.float32).reshape(5, 5)
    u = oracle_mod.unfold(imap, 3)
    assert u[2, 2].tolist() == [6, 7, 8, 11, 12, 13, 16, 17, 18]


def test_unfold_corner_clamps_to_edge(oracle_mod):
    imap = np.arange(25, dtype=np.float32).reshape(5, 5)
    u = oracle_mod.unfold(imap, 3)
    # (0,0): rows {0,0,1}, cols {0,0,1}
    assert u[0, 0].tolist() == [0, 0, 1, 0, 0, 1, 5, 5, 6]
    # (4,2): rows {3,4,4}, cols {1,2,3}
    assert u[4, 2].tolist() == [16, 17, 18, 21, 22, 23, 21, 22, 23]


def test_unfold_k1_and_constant(oracle_mod):
    imap = RNG.standard_normal((6, 7)).astype(np.float32)
    assert np.array_equal(oracle_mod.unfold(imap, 1)[..., 0], imap.astype(np.float64))
    c = np.full((6, 7), 0.375, np.float32)
    assert np.all(oracle_mod.unfold(c, 5) == 0.375)


# ---------------------------------------------------------------- softmax (Eq. 3)
def test_kernel_map_constant_importance_is_uniform(oracle_mod):
    km = oracle_mod.kernel_map(np.full((7, 9), -3.25, np.float32), 3)
    assert np.allclose(km, 1.0 / 9.0, rtol=0, atol=1e-16)


def test_kernel_map_dominant_neighbour(oracle_mod):
    # a neighbour 40 above the rest takes > 1 - 1e-10 of the weight.
    imap = np.zeros((5, 5), np.float32)
    imap[1, 3] = 40.0
    km = oracle_mod.kernel_map(imap, 3)
    # for pixel (2,2), tap (1,3) is offset (-1,+1) -> j = 0*3 + 2 = 2
    assert km[2, 2, 2] > 1 - 1e-10
    # Eq. 3 orientation: the weight follows I(q), not I(p): pixel (1,3)'s own
    # window has the spike at its centre tap j = 4.
    assert km[1, 3, 4] > 1 - 1e-10


def test_kernel_map_matches_closed_form_exp_ratio(oracle_mod):
    imap = RNG.uniform(-3, 3, (6, 8)).astype(np.float32)
    km = oracle_mod.kernel_map(imap, 5)
    assert np.allclose(km.sum(-1), 1.0, rtol=0, atol=1e-14)
    e = np.exp(oracle_mod.unfold(imap, 5))
    assert np.allclose(km, e / e.sum(-1, keepdims=True), rtol=1e-14, atol=0)
    assert km.min() >= 0 and km.max() <= 1


# ------------------------------------------------------------ Eq. 3 + Eq. 4 pins
@pytest.mark.parametrize("k", [1, 3, 5, 7, 13])
def test_uniform_importance_is_scipy_box_filter(oracle_mod, k):
    # Constant I makes every weight 1/k^2, so Eq. 4 is the k x k box mean.
    H, W = 17, 23
    rad = RNG.exponential(1.0, (1, 3, H, W)).astype(np.float32)
    imp = np.full((1, 1, H, W), 1.5, np.float32)
    out = oracle_mod.decode_filter_fuse(rad, imp, None, [k])[0]
    for c in range(3):
        np.testing.assert_allclose(out[c], _box(rad[0, c], k), rtol=1e-13, atol=0)


@pytest.mark.parametrize("k", [3, 5, 9, 13])
def test_ratio_of_box_filters_identity(oracle_mod, k):
    # Eq. 3 weights depend on q only, so R = box(e*r) / box(e), e = exp(I):
    # an independent closed form evaluated with scipy's box filter.
    H, W = 19, 29  # H != W catches transposed dy/dx
    rad = RNG.exponential(1.0, (1, 3, H, W)).astype(np.float32)
    imp = RNG.uniform(-4, 4, (1, 1, H, W)).astype(np.float32)
    out = oracle_mod.decode_filter_fuse(rad, imp, None, [k])[0]
    e = np.exp(imp[0, 0].astype(np.float64))
    den = _box(e, k)
    for c in range(3):
        ref = _box(e * rad[0, c].astype(np.float64), k) / den
        np.testing.assert_allclose(out[c], ref, rtol=1e-12, atol=0)


def test_k1_is_identity_exactly(oracle_mod):
    rad, imp, _ = _rand_inputs(9, 11, 1, RNG)
    out = oracle_mod.decode_filter_fuse(rad, imp, None, [1])
    assert np.array_equal(out.astype(np.float32), rad)


def test_constant_radiance_reproduced_exactly(oracle_mod):
    # sum_q w_p(q) = 1, so a constant image is reproduced (fp64 then fp32 rounding).
    H, W = 14, 15
    rad = np.full((1, 3, H, W), 0.3712, np.float32)
    _, imp, blend = _rand_inputs(H, W, 3, RNG, imp_scale=5.0)
    out = oracle_mod.decode_filter_fuse(rad, imp, blend, [3, 7, 13])
    assert np.array_equal(out.astype(np.float32), rad)


def test_convex_hull_of_window(oracle_mod):
    H, W, k = 12, 13, 5
    rad, imp, _ = _rand_inputs(H, W, 1, RNG, imp_scale=4.0)
    out = oracle_mod.decode_filter_fuse(rad, imp, None, [k])[0]
    from scipy.ndimage import maximum_filter, minimum_filter
    for c in range(3):
        lo = minimum_filter(rad[0, c], size=k, mode="nearest")
        hi = maximum_filter(rad[0, c], size=k, mode="nearest")
        assert np.all(out[c] >= lo * (1 - 1e-15)) and np.all(out[c] <= hi * (1 + 1e-15))


def test_linear_in_radiance_and_shift_invariant_in_importance(oracle_mod):
    H, W = 10, 12
    r1, imp, blend = _rand_inputs(H, W, 2, RNG)
    r2, _, _ = _rand_inputs(H, W, 2, RNG)
    sizes = [3, 5]
    o1 = oracle_mod.decode_filter_fuse(r1, imp, blend, sizes)
    o2 = oracle_mod.decode_filter_fuse(r2, imp, blend, sizes)
    a, b = np.float32(0.75), np.float32(2.0)
    o12 = oracle_mod.decode_filter_fuse(a * r1 + b * r2, imp, blend, sizes)
    # a*r1 + b*r2 is rounded to fp32 once; compare with that tolerance
    np.testing.assert_allclose(o12, 0.75 * o1 + 2.0 * o2, rtol=2e-7)
    # I -> I + const ("a relative value")
    o_shift = oracle_mod.decode_filter_fuse(r1, imp + np.float32(7.0), blend, sizes)
    np.testing.assert_allclose(o_shift, o1, rtol=2e-6)  # I+7 rounds I in fp32
    # logits -> logits + const
    o_lshift = oracle_mod.decode_filter_fuse(r1, imp, blend + np.float32(3.0), sizes)
    np.testing.assert_allclose(o_lshift, o1, rtol=2e-6)


@pytest.mark.parametrize("op", ["flipud", "fliplr", "transpose"])
def test_flip_transpose_equivariance_everywhere(oracle_mod, op):
    # The clamp border is symmetric, so the whole map (borders included) is
    # equivariant under the dihedral symmetries of the grid.
    H, W = 11, 16
    rad, imp, blend = _rand_inputs(H, W, 3, RNG)
    sizes = [3, 5, 9]
    f = {"flipud": lambda a: a[..., ::-1, :], "fliplr": lambda a: a[..., ::-1],
         "transpose": lambda a: np.swapaxes(a, -1, -2)}[op]
    o = oracle_mod.decode_filter_fuse(rad, imp, blend, sizes)
    of = oracle_mod.decode_filter_fuse(f(rad), f(imp), f(blend), sizes)
    np.testing.assert_allclose(of, f(o), rtol=1e-13)


def test_interior_translation_equivariance(oracle_mod):
    H, W, k, s = 24, 24, 5, 3
    rad, imp, _ = _rand_inputs(H, W, 1, RNG)
    o = oracle_mod.decode_filter_fuse(rad, imp, None, [k])[0]
    o_s = oracle_mod.decode_filter_fuse(np.roll(rad, (s, s), (-2, -1)),
                                        np.roll(imp, (s, s), (-2, -1)), None, [k])[0]
    r = k // 2
    inner = np.s_[:, r + s:H - r, r + s:W - r]
    np.testing.assert_allclose(o_s[inner], np.roll(o, (s, s), (-2, -1))[inner], rtol=1e-13)


# ------------------------------------------------------------------ fusion (Eq. 5)
def _filtered(oracle_mod, rad, imp, sizes):
    return np.stack([oracle_mod.decode_filter_fuse(rad, imp[:, i:i + 1], None, [k])[0]
                     for i, k in enumerate(sizes)])


def test_fusion_equal_logits_is_mean_and_dominant_logit_selects(oracle_mod):
    H, W = 13, 14
    sizes = [3, 7, 11]
    rad, imp, _ = _rand_inputs(H, W, 3, RNG)
    Ri = _filtered(oracle_mod, rad, imp, sizes)
    eq = np.zeros((1, 3, H, W), np.float32)
    out = oracle_mod.decode_filter_fuse(rad, imp, eq, sizes)[0]
    np.testing.assert_allclose(out, Ri.mean(0), rtol=1e-14)
    # a dominant logit on map 1 selects R^{k_1} (catches alpha_i paired with R_j)
    dom = np.zeros((1, 3, H, W), np.float32)
    dom[:, 1] = 40.0
    out = oracle_mod.decode_filter_fuse(rad, imp, dom, sizes)[0]
    np.testing.assert_allclose(out, Ri[1], rtol=1e-8)
    # and R^{k_1} itself is the closed-form ratio of box filters for k=7
    e = np.exp(imp[0, 1].astype(np.float64))
    ref = _box(e * rad[0, 0], 7) / _box(e, 7)
    np.testing.assert_allclose(Ri[1][0], ref, rtol=1e-12)


def test_fusion_M1_identity_and_prenormalised_alpha(oracle_mod):
    H, W = 8, 9
    rad, imp, _ = _rand_inputs(H, W, 2, RNG)
    one = oracle_mod.decode_filter_fuse(rad, imp[:, :1], None, [5])
    with_logit = oracle_mod.decode_filter_fuse(rad, imp[:, :1],
                                               np.full((1, 1, H, W), 3.0, np.float32), [5])
    assert np.array_equal(one, with_logit)
    Ri = _filtered(oracle_mod, rad, imp, [3, 5])
    a = RNG.uniform(0, 1, (1, 1, H, W)).astype(np.float32)
    alpha = np.concatenate([a, 1 - a], axis=1).astype(np.float32)
    out = oracle_mod.decode_filter_fuse(rad, imp, alpha, [3, 5], blend_is_logits=False)[0]
    ref = alpha[0, 0].astype(np.float64) * Ri[0] + alpha[0, 1].astype(np.float64) * Ri[1]
    np.testing.assert_allclose(out, ref, rtol=1e-14)


def test_fuse_entry_point_closed_form(oracle_mod):
    H, W, M = 4, 5, 3
    filt = RNG.standard_normal((M, 3, H, W))
    logits = RNG.standard_normal((M, H, W)).astype(np.float32)
    out = oracle_mod.fuse(filt, logits)
    a = np.exp(logits.astype(np.float64))
    a /= a.sum(0)
    np.testing.assert_allclose(out, (a[:, None] * filt).sum(0), rtol=1e-14)


# --------------------------------------------------------- hand-worked golden
def test_hand_worked_3x3_golden(oracle_mod):
    g = json.load(open(os.path.join(HERE, "golden", "hand_worked_3x3.json")))
    H, W = g["H"], g["W"]
    imp = np.stack([np.log(np.array(g["exp_importance_k1"], np.float64)),
                    np.log(np.array(g["exp_importance_k3"], np.float64))]).astype(np.float32)
    red = np.array(g["radiance_R"], np.float32)
    rad = np.stack([red, np.ones((H, W), np.float32), 10 - red])[None]
    blend = np.stack([np.full((H, W), np.log(float(v)), np.float32) for v in g["exp_blend"]])[None]
    out = oracle_mod.decode_filter_fuse(rad, imp[None], blend, g["sizes"])[0]
    k3 = oracle_mod.decode_filter_fuse(rad, imp[None, 1:2], None, [3])[0]
    # the inputs are fp32 roundings of ln(n); the tolerance covers that (~1e-7)
    for key, frac in g["expected_k3_R"].items():
        y, x = eval(key)
        assert k3[0, y, x] == pytest.approx(float(Fraction(frac)), rel=2e-7)
    for key, frac in g["expected_fused_R"].items():
        y, x = eval(key)
        assert out[0, y, x] == pytest.approx(float(Fraction(frac)), rel=2e-7)
        assert out[2, y, x] == pytest.approx(10 - float(Fraction(frac)), rel=2e-7)
    np.testing.assert_allclose(out[1], 1.0, rtol=1e-15)


# ------------------------------------------------------- 50-digit brute force
def _brute(rad, imp, blend, sizes):
    """Eq. 3-5 per (p, q) pair at 50 digits, no max shift, no shared helpers."""
    mpmath.mp.dps = 50
    _, H, W = rad.shape
    M = len(sizes)
    out = np.zeros((3, H, W))
    for y in range(H):
        for x in range(W):
            Rs = []
            for i, k in enumerate(sizes):
                r = k // 2
                taps = [(min(max(y + dy, 0), H - 1), min(max(x + dx, 0), W - 1))
                        for dy in range(-r, r + 1) for dx in range(-r, r + 1)]
                den = mpmath.fsum(mpmath.exp(mpmath.mpf(float(imp[i, qy, qx])))
                                  for qy, qx in taps)
                Rs.append([mpmath.fsum(mpmath.exp(mpmath.mpf(float(imp[i, qy, qx])))
                                       * mpmath.mpf(float(rad[c, qy, qx]))
                                       for qy, qx in taps) / den for c in range(3)])
            if M == 1:
                alpha = [mpmath.mpf(1)]
            else:
                a = [mpmath.exp(mpmath.mpf(float(blend[i, y, x]))) for i in range(M)]
                s = mpmath.fsum(a)
                alpha = [ai / s for ai in a]
            for c in range(3):
                out[c, y, x] = float(mpmath.fsum(alpha[i] * Rs[i][c] for i in range(M)))
    return out


@pytest.mark.parametrize("sizes", [[3], [5, 3], [1, 3, 7], [7, 5, 3]])
def test_brute_force_8x8_mpmath(oracle_mod, sizes):
    rng = np.random.default_rng(len(sizes) * 31 + sizes[0])
    H = W = 8
    rad, imp, blend = _rand_inputs(H, W, len(sizes), rng, imp_scale=3.0)
    out = oracle_mod.decode_filter_fuse(rad, imp, blend if len(sizes) > 1 else None, sizes)[0]
    ref = _brute(rad[0], imp[0], blend[0], sizes)
    np.testing.assert_allclose(out, ref, rtol=1e-13, atol=0)


# --------------------------------------------- internal consistency + API edges
def test_streaming_equals_explicit_and_rows_pixels_agree(oracle_mod):
    H, W = 21, 18
    sizes = [3, 5, 7, 9, 11, 13]
    rad, imp, blend = _rand_inputs(H, W, 6, RNG)
    s = oracle_mod.decode_filter_fuse(rad, imp, blend, sizes)
    e = oracle_mod.explicit_decode_filter_fuse(rad[0], imp[0], blend[0], sizes)
    np.testing.assert_allclose(s[0], e, rtol=1e-14)
    rows = oracle_mod.decode_filter_fuse(rad, imp, blend, sizes, rows=(5, 12))
    assert np.array_equal(rows, s[:, :, 5:12])
    ys, xs = np.array([0, 20, 7]), np.array([17, 0, 9])
    px = oracle_mod.decode_filter_fuse_pixels(rad, imp, blend, sizes, [0, 0, 0], ys, xs)
    assert np.array_equal(px, s[0][:, ys, xs].T)


def test_oracle_rejects_bad_config(oracle_mod):
    rad, imp, blend = _rand_inputs(6, 6, 2, RNG)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.decode_filter_fuse(rad, imp, blend, [3, 4])      # even k
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.decode_filter_fuse(rad, imp, blend, [3, 7])      # k > min(H,W)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.decode_filter_fuse(rad, imp, None, [3, 5])       # M > 1 needs blend


def test_softmax_stays_finite_for_huge_importance(oracle_mod):
    # DESIGN.md R2: the max-shifted softmax equals Eq. 3 exactly and stays
    # finite where exp(I) itself would overflow (exp(1000) = inf in fp64).
    imap = np.full((5, 5), -1000.0, np.float32)
    imap[4, 4] = 1000.0       # the last tap (j = 8) of pixel (3,3)'s window
    km = oracle_mod.kernel_map(imap, 3)
    assert np.all(np.isfinite(km))
    np.testing.assert_allclose(km.sum(-1), 1.0, rtol=0, atol=1e-15)
    assert km[3, 3, 8] == 1.0 and km[0, 0, 0] == pytest.approx(1 / 9, rel=1e-15)


# ------------------------------------------- albedo demod/remod (NEXT row 1)
def test_demodulate_remodulate_spec_examples(oracle_mod):
    # SPEC.md:132-135 and 141-144 examples
    r = np.array([0.6, 0.001, 2.0], np.float32)
    a = np.array([0.3, 0.0, 1.0], np.float32)
    d = oracle_mod.demodulate(r, a, eps=1e-3)
    assert d[0] == pytest.approx(2.0, rel=1e-7)      # 0.6 / 0.3 (fp32 inputs)
    assert d[1] == pytest.approx(1.0, rel=1e-7)      # eps floor: 0.001 / 1e-3
    assert d[2] == 2.0                               # albedo 1 -> identity
    m = oracle_mod.remodulate(np.array([2.0, 5.0]), np.array([0.3, 1.0], np.float32))
    assert m[0] == pytest.approx(0.6, rel=1e-7) and m[1] == 5.0


def test_demod_remod_round_trip(oracle_mod):
    # remodulate(demodulate(r)) = r wherever albedo >= eps
    rng = np.random.default_rng(3)
    r = rng.exponential(1.0, 1000).astype(np.float32)
    a = rng.uniform(0.01, 1.0, 1000).astype(np.float32)
    back = oracle_mod.remodulate(oracle_mod.demodulate(r, a, 1e-3), a)
    np.testing.assert_allclose(back, r.astype(np.float64), rtol=1e-15)


# ---------------------------------------- multi-resolution "Ours MR" (NEXT row 2)
def test_downsample_upsample_spec_examples(oracle_mod):
    # [1,2,3,4] -> 2.5; constant -> constant; block mean brute force
    assert oracle_mod.downsample_2x2(np.array([[1, 2], [3, 4]], np.float32))[0, 0] == 2.5
    c = np.full((6, 8), 0.75, np.float32)
    assert np.all(oracle_mod.downsample_2x2(c) == 0.75)
    x = RNG.standard_normal((2, 8, 10)).astype(np.float32)
    ref = x.astype(np.float64).reshape(2, 4, 2, 5, 2).mean(axis=(2, 4))
    np.testing.assert_allclose(oracle_mod.downsample_2x2(x), ref, rtol=1e-15, atol=1e-15)
    # U replicates; U(D(constant)) = identity; min/max preserved
    u = oracle_mod.upsample_nearest(np.array([[7.0]]))
    assert u.shape == (2, 2) and np.all(u == 7.0)
    y = RNG.standard_normal((3, 4, 5))
    uy = oracle_mod.upsample_nearest(y)
    assert np.array_equal(uy[:, ::2, ::2], y) and np.array_equal(uy[:, 1::2, 1::2], y)


def test_combine_resolutions_spec_examples(oracle_mod):
    # SPEC.md:303-306 / Eq. 7
    N, H, W = 1, 8, 6
    fine = RNG.exponential(1.0, (N, 3, H, W))
    coarse = RNG.exponential(1.0, (N, 3, H // 2, W // 2))
    zero = np.zeros((N, 1, H, W), np.float32)
    assert np.array_equal(oracle_mod.combine_resolutions(fine, coarse, zero), fine)   # alpha = 0
    a = RNG.uniform(0, 1, (N, 1, H, W)).astype(np.float32)
    dfine = oracle_mod.downsample_2x2(fine.astype(np.float32)).astype(np.float64)
    f32 = fine.astype(np.float32).astype(np.float64)
    np.testing.assert_allclose(oracle_mod.combine_resolutions(f32, dfine, a), f32, rtol=1e-15)  # coarse = D(fine)
    one = np.ones((N, 1, H, W), np.float32)
    out = oracle_mod.combine_resolutions(np.full((N, 3, H, W), 2.0), np.full((N, 3, H // 2, W // 2), 5.0), one)
    assert np.all(out == 5.0)                                                           # alpha = 1, constants


def test_mr_single_level_is_plain_decoder(oracle_mod):
    rad, imp, blend = _rand_inputs(8, 12, 2, RNG)
    a = oracle_mod.mr_decode_filter_fuse(rad, [imp], [blend], [], [[3, 5]])
    b = oracle_mod.decode_filter_fuse(rad, imp, blend, [3, 5])
    assert np.array_equal(a, b)


def _mr_level_inputs(H, W, sizes, rng):
    imps, blends = [], []
    for l, s in enumerate(sizes):
        _, i, b = _rand_inputs(H >> l, W >> l, len(s), rng)
        imps.append(i)
        blends.append(b)
    return imps, blends


def test_mr_three_levels_alpha_zero_is_level0_decoder(oracle_mod):
    # Eq. 7 with alpha = 0 everywhere: o = f at every level, so the output is
    # level 0's plain decoder (reading R18)
    H, W, sizes = 24, 32, [[3, 5], [3, 5], [3, 5]]
    rad, _, _ = _rand_inputs(H, W, 1, RNG)
    imps, blends = _mr_level_inputs(H, W, sizes, RNG)
    alphas = [np.zeros((1, 1, H >> l, W >> l), np.float32) for l in range(2)]
    a = oracle_mod.mr_decode_filter_fuse(rad, imps, blends, alphas, sizes)
    b = oracle_mod.decode_filter_fuse(rad, imps[0], blends[0], sizes[0])
    assert np.array_equal(a, b)


def test_mr_three_levels_constant_radiance_exact(oracle_mod):
    # every level reproduces a constant (to fp64 rounding, exactly after fp32
    # rounding) and D, U keep it, so f + alpha (U c - U D f) = K for any alpha
    H, W, sizes = 24, 32, [[3, 5], [3, 7], [5, 3]]
    rad = np.full((1, 3, H, W), 0.375, np.float32)
    imps, blends = _mr_level_inputs(H, W, sizes, RNG)
    alphas = [RNG.uniform(0, 1, (1, 1, H >> l, W >> l)).astype(np.float32) for l in range(2)]
    out = oracle_mod.mr_decode_filter_fuse(rad, imps, blends, alphas, sizes)
    np.testing.assert_allclose(out, 0.375, rtol=1e-14, atol=0)
    assert np.all(out.astype(np.float32) == np.float32(0.375))


def test_mr_two_levels_uniform_importance_is_scipy_pyramid(oracle_mod):
    # Uniform importance turns every level into a clamp-to-edge box mean
    # (pinned above), so a two-level M = 1 "Ours MR" is, written with scipy and
    # numpy only: f = box_3(r), c = box_5(D r) (D r in fp64), o = f + a (U c - U D f)
    H, W = 12, 20
    rad = RNG.exponential(1.0, (1, 3, H, W)).astype(np.float32)
    imps = [np.zeros((1, 1, H, W), np.float32), np.zeros((1, 1, H // 2, W // 2), np.float32)]
    alpha = RNG.uniform(0, 1, (1, 1, H, W)).astype(np.float32)
    out = oracle_mod.mr_decode_filter_fuse(rad, imps, None, [alpha], [[3], [5]])

    def D(x):
        return x.reshape(x.shape[0], x.shape[1], x.shape[2] // 2, 2, x.shape[3] // 2, 2).mean(axis=(3, 5))

    def U(x):
        return np.repeat(np.repeat(x, 2, axis=2), 2, axis=3)

    r64 = rad.astype(np.float64)
    f = np.stack([_box(r64[0, c], 3) for c in range(3)])[None]
    dr = D(r64)
    cc = np.stack([_box(dr[0, c], 5) for c in range(3)])[None]
    ref = f + alpha.astype(np.float64) * (U(cc) - U(D(f)))
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------ backward (NEXT row 3)
def _torch_forward_fp64(rad, imp, blend, sizes, logits=True):
    """Eq. 3-5 written with torch library steps (replicate pad + F.unfold,
    softmax), independent of the C oracle's loops; autograd differentiates it."""
    import torch
    import torch.nn.functional as F
    N, _, H, W = rad.shape
    out = 0.0
    Rs = []
    for i, k in enumerate(sizes):
        r = (k - 1) // 2
        Ii = F.pad(imp[:, i:i + 1], (r, r, r, r), mode="replicate")
        rp = F.pad(rad, (r, r, r, r), mode="replicate")
        u = F.unfold(Ii, k).view(N, 1, k * k, H, W)
        w = torch.softmax(u, dim=2)
        v = F.unfold(rp, k).view(N, 3, k * k, H, W)
        Rs.append((w * v).sum(dim=2))
    if len(sizes) == 1:
        return Rs[0]
    a = torch.softmax(blend, dim=1) if logits else blend
    for i, R in enumerate(Rs):
        out = out + a[:, i:i + 1] * R
    return out


@pytest.mark.parametrize("sizes,logits", [((3, 5), True), ((5,), True), ((3, 5, 7), False)])
def test_backward_matches_autograd_of_library_forward(oracle_mod, sizes, logits):
    # pin: torch autograd of an unfold/softmax forward in fp64 (Eq. 1:
    # the decoder is trained end to end, so its gradients are those of Eq. 3-5).
    import torch
    rng = np.random.default_rng(31)
    M = len(sizes)
    rad, imp, blend = _rand_inputs(9, 11, M, rng)
    if not logits:
        blend = rng.uniform(0, 1, size=blend.shape).astype(np.float32)
    G = rng.standard_normal((1, 3, 9, 11))
    gI, gB = oracle_mod.backward(rad, imp, blend, G, sizes, blend_is_logits=logits)
    ti = torch.tensor(imp, dtype=torch.float64, requires_grad=True)
    tb = torch.tensor(blend, dtype=torch.float64, requires_grad=True)
    out = _torch_forward_fp64(torch.tensor(rad, dtype=torch.float64), ti, tb, sizes, logits)
    (out * torch.tensor(G)).sum().backward()
    np.testing.assert_allclose(gI, ti.grad.numpy(), rtol=1e-10, atol=1e-12)
    if M > 1:
        np.testing.assert_allclose(gB, tb.grad.numpy(), rtol=1e-10, atol=1e-12)
    else:
        assert np.all(gB == 0)


def test_backward_central_differences(oracle_mod):
    # pin: central differences of the (pinned) fp64 forward with exactly
    # representable perturbations (inputs on a 2^-12 grid, h = 2^-10).
    rng = np.random.default_rng(32)
    sizes = (3, 5)
    rad, imp, blend = _rand_inputs(6, 7, 2, rng)
    imp = (np.round(imp * 4096) / 4096).astype(np.float32)
    blend = (np.round(blend * 4096) / 4096).astype(np.float32)
    G = rng.standard_normal((1, 3, 6, 7))
    gI, gB = oracle_mod.backward(rad, imp, blend, G, sizes)
    h = 2.0 ** -10

    def L(im, bl):
        return float((oracle_mod.decode_filter_fuse(rad, im, bl, sizes) * G).sum())

    for arr, grad, which in ((imp, gI, 0), (blend, gB, 1)):
        fd = np.zeros_like(grad)
        for idx in np.ndindex(arr.shape):
            p, m = arr.copy(), arr.copy()
            p[idx] += np.float32(h)
            m[idx] -= np.float32(h)
            lp = L(p, blend) if which == 0 else L(imp, p)
            lm = L(m, blend) if which == 0 else L(imp, m)
            fd[idx] = (lp - lm) / (2 * h)
        np.testing.assert_allclose(grad, fd, rtol=0, atol=2e-5 * np.abs(fd).max())


def test_backward_invariants(oracle_mod):
    # shift invariance of Eq. 3 in I_i and of Eq. 5 in B: gradients sum to 0;
    # constant radiance makes every R_i the same constant -> dL/dI = 0 and dL/dB = 0
    # (SPEC.md:296); grad_out = 0 -> all zero.
    rng = np.random.default_rng(33)
    sizes = (3, 5, 7)
    rad, imp, blend = _rand_inputs(10, 12, 3, rng)
    G = rng.standard_normal((1, 3, 10, 12))
    gI, gB = oracle_mod.backward(rad, imp, blend, G, sizes)
    scale = np.abs(gI).max()
    assert scale > 0
    assert np.abs(gI.sum(axis=(2, 3))).max() < 1e-12 * scale * gI[0, 0].size
    assert np.abs(gB.sum(axis=1)).max() < 1e-14 * max(1.0, np.abs(gB).max()) * 10
    crad = np.full_like(rad, 0.625)
    gI0, gB0 = oracle_mod.backward(crad, imp, blend, G, sizes)
    assert np.abs(gI0).max() < 1e-14 and np.abs(gB0).max() < 1e-14
    gI1, gB1 = oracle_mod.backward(rad, imp, blend, np.zeros_like(G), sizes)
    assert np.all(gI1 == 0) and np.all(gB1 == 0)


# ------------------------------------------ temporal accumulation (NEXT row 4)
def _temporal_case(rng, H=7, W=9, N=1):
    rad = rng.exponential(1.0, size=(N, 3, H, W)).astype(np.float32)
    prev = rng.exponential(1.0, size=(N, 3, H, W)).astype(np.float32)
    pos = (10 * rng.standard_normal((N, 3, H, W))).astype(np.float32)
    nrm = rng.uniform(0, 1, size=(N, 3, H, W)).astype(np.float32)
    valid = np.ones((N, H, W), np.uint8)
    motion = np.zeros((N, 2, H, W), np.float32)
    return rad, prev, pos, nrm, valid, motion


def test_temporal_zero_motion_identical_geometry(oracle_mod):
    # SPEC.md:152-153 (identity warp) and :160 (identical geometry passes):
    # accum = (1 - a) prev + a cur everywhere
    rng = np.random.default_rng(41)
    rad, prev, pos, nrm, valid, motion = _temporal_case(rng)
    nrm = np.where(np.abs(2 * nrm - 1).sum(axis=1, keepdims=True) < 0.2, 0.9, nrm).astype(np.float32)
    acc, mask = oracle_mod.temporal_accumulate(rad, prev, pos, nrm, valid, pos, nrm, motion, pos_tol=0.5,
                                               normal_tol=0.9, alpha=0.25)
    assert mask.all()
    np.testing.assert_allclose(acc, 0.75 * prev.astype(np.float64) + 0.25 * rad, rtol=1e-15)


def test_temporal_out_of_bounds_keeps_current_exactly(oracle_mod):
    # SPEC.md:154 motion (+W, 0) -> mask all false; §4.1 "failed pixels
    # remain original 1 spp": accum == cur bit for bit; NaN motion likewise
    rng = np.random.default_rng(42)
    rad, prev, pos, nrm, valid, motion = _temporal_case(rng)
    motion[:, 0] = rad.shape[3]
    acc, mask = oracle_mod.temporal_accumulate(rad, prev, pos, nrm, valid, pos, nrm, motion, pos_tol=1e3)
    assert not mask.any() and np.array_equal(acc, rad.astype(np.float64))
    motion[:, 0] = np.nan
    acc, mask = oracle_mod.temporal_accumulate(rad, prev, pos, nrm, valid, pos, nrm, motion, pos_tol=1e3)
    assert not mask.any() and np.array_equal(acc, rad.astype(np.float64))


def test_temporal_integer_shift(oracle_mod):
    # shift (1, 0): warped(i, j) = prev(i, j+1) where in bounds.
    # With cur = 0 the accumulation is (1 - a) warped, so warped is read back.
    rng = np.random.default_rng(43)
    rad, prev, pos, nrm, valid, motion = _temporal_case(rng, H=6, W=8)
    motion[:, 0] = 1.0
    cur = np.zeros_like(rad)
    acc, mask = oracle_mod.temporal_accumulate(cur, prev, pos, nrm, valid, pos, nrm, motion, pos_tol=1e6,
                                               normal_tol=1e-6, alpha=0.5)
    # geometry test uses prev(i, j+1) vs cur(i, j): disable it with huge tolerances,
    # except normals: compare only where the shifted normals pass
    W = rad.shape[3]
    assert not mask[..., W - 1].any()
    sel = mask[..., : W - 1].astype(bool)
    assert sel.any()
    warped = acc[:, :, :, : W - 1] / 0.5
    ref = prev[:, :, :, 1:].astype(np.float64)
    np.testing.assert_array_equal(warped[np.broadcast_to(sel[:, None], warped.shape)],
                                  ref[np.broadcast_to(sel[:, None], ref.shape)])


def test_temporal_nearest_rounding(oracle_mod):
    # nearest pixel of x + m is floor(x + m + 0.5) (reading R21): m = 0.49 stays,
    # m = 0.5 moves, m = -0.5 stays, m = -0.51 moves
    rng = np.random.default_rng(44)
    rad, prev, pos, nrm, valid, motion = _temporal_case(rng, H=3, W=5)
    cur = np.zeros_like(rad)
    for m, shift in ((0.49, 0), (0.5, 1), (-0.5, 0), (-0.51, -1)):
        motion[:, 0] = m
        acc, mask = oracle_mod.temporal_accumulate(cur, prev, pos, nrm, valid, pos, nrm, motion, pos_tol=1e6,
                                                   normal_tol=1e-6, alpha=0.5)
        j = 2
        if mask[0, 1, j]:
            assert acc[0, 0, 1, j] == 0.5 * prev[0, 0, 1, j + shift]


def test_temporal_consistency_thresholds(oracle_mod):
    # displaced positions (10 x tol) fail; flipped normals fail;
    # invalid history fails; blend arithmetic 0.2: warped 1, cur 0 -> 0.8
    H, W = 4, 5
    one = np.ones((1, 3, H, W), np.float32)
    pos = np.zeros((1, 3, H, W), np.float32)
    nrm = np.full((1, 3, H, W), 1.0, np.float32)   # (1,1,1) after un-scaling
    valid = np.ones((1, H, W), np.uint8)
    motion = np.zeros((1, 2, H, W), np.float32)
    acc, mask = oracle_mod.temporal_accumulate(0 * one, one, pos, nrm, valid, pos, nrm, motion, pos_tol=0.1,
                                               alpha=0.2)
    assert mask.all()
    np.testing.assert_allclose(acc, 0.8, rtol=1e-7)  # alpha is the fp32 value of 0.2
    far = pos.copy(); far[:, 2] = 1.0
    _, mask = oracle_mod.temporal_accumulate(0 * one, one, pos, nrm, valid, far, nrm, motion, pos_tol=0.1)
    assert not mask.any()
    _, mask = oracle_mod.temporal_accumulate(0 * one, one, pos, nrm, valid, pos, 1 - nrm, motion, pos_tol=0.1)
    assert not mask.any()
    v2 = valid.copy(); v2[0, 1, 2] = 0
    _, mask = oracle_mod.temporal_accumulate(0 * one, one, pos, nrm, v2, pos, nrm, motion, pos_tol=0.1)
    assert mask.sum() == H * W - 1 and mask[0, 1, 2] == 0


def test_temporal_alpha_one_is_identity_and_mask_matches_predicates(oracle_mod):
    # SPEC.md invariants: alpha = 1 -> output = cur regardless of the mask;
    # random buffers: mask equals a direct float32 evaluation of both predicates
    rng = np.random.default_rng(45)
    rad, prev, pos, nrm, valid, motion = _temporal_case(rng, H=16, W=20)
    cpos = (pos + rng.standard_normal(pos.shape).astype(np.float32)).astype(np.float32)
    cnrm = np.clip(nrm + 0.3 * rng.standard_normal(nrm.shape), 0, 1).astype(np.float32)
    acc, mask = oracle_mod.temporal_accumulate(rad, prev, pos, nrm, valid, cpos, cnrm, motion, pos_tol=1.5,
                                               normal_tol=0.8, alpha=1.0)
    assert np.array_equal(acc, rad.astype(np.float64))
    f = np.float32
    d = (cpos - pos).astype(f)
    d2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
    a = (f(2) * cnrm - f(1)).astype(f)
    b = (f(2) * nrm - f(1)).astype(f)
    dot = (a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1]) + a[:, 2] * b[:, 2]
    aa = (a[:, 0] * a[:, 0] + a[:, 1] * a[:, 1]) + a[:, 2] * a[:, 2]
    bb = (b[:, 0] * b[:, 0] + b[:, 1] * b[:, 1]) + b[:, 2] * b[:, 2]
    ref = (d2 < f(1.5) * f(1.5)) & (dot > f(0.8) * np.sqrt(aa * bb))
    assert 0.05 < ref.mean() < 0.95
    assert np.array_equal(mask.astype(bool), ref)


def test_temporal_reduces_variance_static_scene(oracle_mod):
    # SPEC.md:172 property: static scene, constant signal c with zero-mean
    # noise; after n accumulated frames the variance is below the input's
    # (EMA with alpha 0.2: asymptotically alpha / (2 - alpha) = 0.11 of it)
    rng = np.random.default_rng(46)
    H, W, c = 48, 48, 2.0
    pos = np.zeros((1, 3, H, W), np.float32)
    nrm = np.full((1, 3, H, W), 0.9, np.float32)
    valid = np.ones((1, H, W), np.uint8)
    motion = np.zeros((1, 2, H, W), np.float32)
    acc = (c + rng.standard_normal((1, 3, H, W))).astype(np.float32)
    for _ in range(30):
        cur = (c + rng.standard_normal((1, 3, H, W))).astype(np.float32)
        acc, _ = oracle_mod.temporal_accumulate(cur, acc.astype(np.float32), pos, nrm, valid, pos, nrm, motion,
                                                pos_tol=0.1, alpha=0.2)
    v = acc.var()
    assert v < 0.2 and abs(acc.mean() - c) < 0.05


# ----------------------------------------- Eq. 5 through the kmdo_fuse entry point
def test_fuse_entry_point_special_cases(oracle_mod):
    # kmdo_fuse itself (not via decode_filter_fuse): M = 1 is the identity
    # (SPEC.md:275), equal logits give the arithmetic mean, a
    # logit 40 above the others selects its input, and adding a
    # constant to every logit changes nothing.  Inputs differ per
    # (size, channel, pixel) so a wrong index pairs the wrong values.
    M, H, W = 4, 5, 7
    filt = RNG.uniform(0.1, 10.0, (M, 3, H, W))
    np.testing.assert_array_equal(oracle_mod.fuse(filt[:1], None), filt[0])
    np.testing.assert_allclose(oracle_mod.fuse(filt, np.full((M, H, W), 1.25, np.float32)),
                               filt.mean(axis=0), rtol=1e-14)
    for i in range(M):
        b = np.zeros((M, H, W), np.float32)
        b[i] = 40.0
        np.testing.assert_allclose(oracle_mod.fuse(filt, b), filt[i], rtol=1e-15)  # other weights ~ e^-40
    logits = RNG.standard_normal((M, H, W)).astype(np.float32)
    np.testing.assert_allclose(oracle_mod.fuse(filt, logits + np.float32(16.0)), oracle_mod.fuse(filt, logits),
                               rtol=1e-6)
    # alpha given (blend_is_logits=0): the weighted sum with the given weights
    a = RNG.uniform(0, 1, (M, H, W)).astype(np.float32)
    ref = (a.astype(np.float64)[:, None] * filt).sum(axis=0)
    np.testing.assert_allclose(oracle_mod.fuse(filt, a, blend_is_logits=False), ref, rtol=1e-14)


def test_f64_radiance_entry_point_matches_fp32_entry(oracle_mod):
    # the multi-resolution oracle filters fp64 pyramid levels through
    # kmdo_decode_filter_fuse_rows_f64rad: on fp32-representable values it must
    # return exactly what the fp32 entry point returns
    rad, imp, blend = _rand_inputs(9, 12, 2, RNG)
    a = oracle_mod.decode_filter_fuse(rad, imp, blend, [3, 5])
    b = oracle_mod.decode_filter_fuse(rad.astype(np.float64), imp, blend, [3, 5])
    np.testing.assert_array_equal(a, b)
