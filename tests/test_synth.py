"""Synthetic scene generators: the reference recipe and the counter hash whose
device kernel and numpy twin must agree bit for bit."""

import numpy as np
import pytest

from paper_1803_00737_b200 import synth


def test_reference_recipe_shapes():
    """bench.py:39-47"""
    pan, ms = synth.synth_scene(64, 32, bands=3, seed=42)
    assert pan.shape == (32, 64) and pan.dtype == np.float32
    assert len(ms) == 3 and all(b.shape == (16, 32) and b.dtype == np.float32 for b in ms)
    again, _ = synth.synth_scene(64, 32, bands=3, seed=42)
    assert np.array_equal(pan, again)


def test_hash_plane_properties():
    v = synth.hash_plane(42, 0, np.arange(100), np.arange(300))
    assert v.dtype == np.float32 and v.shape == (100, 300)
    assert v.min() >= 0.0 and v.max() < 255.0
    assert abs(float(v.mean()) - 127.5) < 2.0
    w = synth.hash_plane(42, 0, np.arange(50, 60), np.arange(100, 110))
    assert np.array_equal(w, v[50:60, 100:110])  # addressable
    assert not np.array_equal(v, synth.hash_plane(42, 1, np.arange(100), np.arange(300)))
    assert not np.array_equal(v, synth.hash_plane(43, 0, np.arange(100), np.arange(300)))


@pytest.mark.gpu
def test_device_plane_equals_numpy_twin():
    import torch

    t = torch.empty((70, 1030), device="cuda")
    synth.device_plane(t, 42, 3, row0=65000, col0=64000)
    want = synth.hash_plane(42, 3, np.arange(65000, 65070), np.arange(64000, 65030))
    assert np.array_equal(t.cpu().numpy(), want)
