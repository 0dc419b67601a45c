"""The tiled multi-process oracle harness (tests/fullsize.py) reproduces the whole-image oracle:
bands of rows evaluated on crops with an r-row halo give the same out / den / fallback as one
bf_box over the full image (fp64 rounding of the SAT only), so the full-size parity tests
compare against the oracle itself, not an approximation of it."""
import numpy as np

from oracle import bf, fit
from synth import CONFIGS, config_input, config_params

from fullsize import oracle_banded, summarise


def test_banded_oracle_equals_whole_image_oracle():
    spec = CONFIGS["cfg1"]
    params = dict(config_params(spec), radius=9, sigma_s=3.0)
    img = config_input(spec, H=157, W=64)
    out_b, cond_b, fb_b = oracle_banded(img, params, n_workers=2, n_bands=5)
    plan = fit.make_plan(**params)
    out, num, den, fb = bf.bf_box(img, plan, return_parts=True)
    mass = bf.spatial_filter(np.ones(img.shape), plan.sp.boxes)
    assert np.max(np.abs(out_b - out)) <= 1e-9
    assert np.max(np.abs(cond_b - den / mass)) <= 1e-6
    assert np.array_equal(fb_b, fb)


def test_summary_counts_fallbacks_and_worst_pixels():
    ref = np.full((4, 5), 100.0)
    img = np.full((4, 5), 7.0, dtype=np.float32)
    got = ref.copy()
    got[1, 2] += 2e-4
    fb = np.zeros((4, 5), dtype=bool)
    fb[3, 4] = True
    ref[3, 4] = 7.0
    got[3, 4] = 7.0
    cond = np.ones((4, 5), dtype=np.float32)
    cond[3, 4] = -0.01
    s = summarise(got, ref, cond, fb, 255.0, img)
    assert s["pass"] and s["worst"][0]["y"] == 1 and s["worst"][0]["x"] == 2
    assert s["n_oracle_fallbacks"] == 1 and s["n_fallback_match"] == 1
    assert s["worst_conditioned"][0]["cond"] < 0
    got[3, 4] = 8.0
    s = summarise(got, ref, cond, fb, 255.0, img)
    assert not s["pass"] and s["n_fallback_match"] == 0
