"""Synthetic inputs of BASELINE.json's configs (host-side numpy, fixed seeds).

These are stand-ins for the reference's benchmark data:
seeded synthetic arrays with the stated shapes, sizes and value
distributions. They are generated once on the host and consumed identically
by the GPU engine and by the CPU baselines. Arrays are returned as
(M samples, N channels), the reference's MultiSignal orientation.
"""
from __future__ import annotations

import math

import numpy as np

PICKUP_MASK = np.array([[1, 1, 0, 1, 0, 0], [1, 1, 1, 0, 1, 0], [1, 1, 1, 1, 1, 1], [1, 0, 1, 1, 0, 1]])
PICKUP_FREQS = (32.0, 16.0, 8.0, 2.0)
TWO_PI = 6.283185307179586476925286766559


def pickup_signals(n: int = 1000, fs: float = 1000.0) -> np.ndarray:
    """Configs 1-3: synth.cpp:26-45 with the standard mask (libm sin, same order)."""
    out = np.zeros((n, 6))
    for j in range(6):
        for i in range(4):
            if not PICKUP_MASK[i, j]:
                continue
            f = PICKUP_FREQS[i]
            out[:, j] += np.array([math.sin(TWO_PI * f * float(k) / fs) for k in range(n)])
    return out


def image_batch(n_images: int = 256, rows: int = 112, cols: int = 92, seed: int = 2106) -> np.ndarray:
    """Config 4: grayscale images in [0, 255]; 3 gratings (periods 4/12/40 px), 5 blobs, N(0, 5).

    Returned as a (cols, rows * n_images) MultiSignal: every image ROW is a
    channel (row-serialized, image-then-row order), M = 92 samples per channel.
    """
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:rows, 0:cols].astype(np.float64)
    imgs = np.empty((n_images, rows, cols))
    for b in range(n_images):
        img = np.full((rows, cols), rng.uniform(60.0, 160.0))
        for period in (4.0, 12.0, 40.0):
            th = rng.uniform(0.0, math.pi)
            amp = rng.uniform(10.0, 60.0)
            ph = rng.uniform(0.0, TWO_PI)
            img += amp * np.sin(TWO_PI * (xx * math.cos(th) + yy * math.sin(th)) / period + ph)
        for _ in range(5):
            cy, cx = rng.uniform(0, rows), rng.uniform(0, cols)
            sg = rng.uniform(5.0, 20.0)
            amp = rng.uniform(-60.0, 60.0)
            img += amp * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2.0 * sg * sg))
        img += rng.normal(0.0, 5.0, size=(rows, cols))
        imgs[b] = np.clip(img, 0.0, 255.0)
    # channel (b, r) = imgs[b, r, :]  -> (cols, n_images*rows)
    return np.ascontiguousarray(imgs.reshape(n_images * rows, cols).T)


def sine_variates(n_var: int = 4096, n_samp: int = 4096, fs: float = 4096.0, seed: int = 2106) -> np.ndarray:
    """Config 5: each variate = 4 sines (freq log-uniform 1-500 Hz, amp U(0.2,1), phase U(0,2pi)) + N(0, 0.05)."""
    rng = np.random.default_rng(seed)
    t = np.arange(n_samp, dtype=np.float64) / fs
    out = np.empty((n_samp, n_var))
    for j in range(n_var):
        f = np.exp(rng.uniform(math.log(1.0), math.log(500.0), size=4))
        a = rng.uniform(0.2, 1.0, size=4)
        p = rng.uniform(0.0, TWO_PI, size=4)
        x = (a[:, None] * np.sin(TWO_PI * f[:, None] * t[None, :] + p[:, None])).sum(axis=0)
        out[:, j] = x + rng.normal(0.0, 0.05, size=n_samp)
    return out


def serialized_length(M: int, N: int, D: int) -> int:
    return M * N + D * (N - 1)


CONFIGS = {
    "c1": dict(name="serial-EMD pick-up 6x1000 D=50", algo="emd", D=50, max_sift_iters=1000, max_imfs=0, nr=1),
    "c2": dict(name="serial-EEMD pick-up 6x1000 D=50 NR=100", algo="eemd", D=50, max_sift_iters=300, max_imfs=10,
               nr=100),
    "c3": dict(name="serial-CEEMDAN pick-up 6x1000 D=50 NR=500", algo="ceemdan", D=50, max_sift_iters=5000,
               max_imfs=0, nr=500),
    "c4": dict(name="serial-EEMD 256 images 112x92 row-serialized D=10 NR=100", algo="eemd", D=10,
               max_sift_iters=300, max_imfs=0, nr=100),
    "c5": dict(name="serial-EEMD 4096x4096 D=64 NR=1000", algo="eemd", D=64, max_sift_iters=300, max_imfs=0,
               nr=1000),
}


def config_input(key: str) -> np.ndarray:
    if key in ("c1", "c2", "c3"):
        return pickup_signals()
    if key == "c4":
        return image_batch()
    if key == "c5":
        return sine_variates()
    raise KeyError(key)
