"""BASELINE.json workload inputs (initial densities, keyframes) -- CPU.

The keyframe blur is checked against scipy.ndimage.gaussian_filter (sigma 1
cell, reflect, truncate 4: the recipe SURVEY.md §8d names); shapes, support
and non-negativity (KeyframeSet rejects negatives, ao.py:40-41) per config.
"""

import numpy as np
import pytest
import torch
from scipy import ndimage

from paper_1608_01102_b200 import workloads


def test_blur_matches_scipy_gaussian_filter():
    rng = np.random.default_rng(0)
    for shape in [(17, 23), (9, 11, 13)]:
        x = rng.standard_normal(shape)
        got = workloads.blur(torch.from_numpy(x), 1.0).numpy()
        want = ndimage.gaussian_filter(x, 1.0, mode="reflect", truncate=4.0)
        assert np.max(np.abs(got - want)) <= 1e-13


@pytest.mark.parametrize("index", [1, 2, 3, 4, 5])
def test_keyframes_follow_baseline(index):
    w = workloads.config(index)
    if index == 5:   # 128^3: check the generator on the config's recipe at 32^3
        w = workloads.Workload(5, 3, 32, 80, w.dtype, 2, w.K, w.r, "cfg5 recipe at 32^3")
    kf = workloads.keyframes(w, device="cpu")
    want_t = {1: [16], 2: [40], 3: [30, 60], 4: [60], 5: [20, 40, 60, 80]}[index]
    assert sorted(kf) == want_t
    for t, k in kf.items():
        assert tuple(k.shape) == tuple(w.spec.res)
        assert float(k.min()) >= 0.0 and 0.5 < float(k.max()) <= 1.0 + 1e-12
    rho0 = workloads.initial_density(w, device="cpu")
    assert float(rho0.min()) >= 0.0 and tuple(rho0.shape) == tuple(w.spec.res)


def test_cfg1_disc_and_cfg2_letter_f():
    w1 = workloads.config(1)
    k1 = workloads.keyframes(w1, device="cpu")[16].numpy()
    h = w1.spec.h
    x = (np.arange(32) + 0.5) * h
    X, Y = np.meshgrid(x, x, indexing="ij")
    d = np.hypot(X - 0.5, Y - 0.7)
    assert np.all(k1[d <= 0.15 - h] == 1.0) and np.all(k1[d >= 0.15 + h] == 0.0)
    w2 = workloads.config(2)
    k2 = workloads.keyframes(w2, device="cpu")[40].numpy()
    x = (np.arange(128) + 0.5) / 128
    i = lambda v: int(np.argmin(np.abs(x - v)))
    assert k2[i(0.40), i(0.55)] > 0.9      # vertical bar
    assert k2[i(0.65), i(0.75)] > 0.9      # top bar
    assert k2[i(0.55), i(0.54)] > 0.5      # middle bar
    assert k2[i(0.55), i(0.40)] < 1e-3     # outside the F
