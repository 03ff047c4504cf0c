"""Synthetic inputs for the BASELINE configs (no public dataset is used).

Cores follow synthetic.hpp:16-29 (random_factors: one GaussianSampler stream,
cores in order, flat (r, i, s) fill, times `scale`); the draws come from the
library's own counter-based generator (trg_omega), which reproduces the
reference stream exactly. X = reconstruct_full(cores) is evaluated on the
device, then optional [0,1] rescaling and noise at an exact SNR
(SPEC.md:338-346). Seeds: cores S, noise S+1, spec.seed = cfg.seed = S, S = 0.

C4 is the builder-defined stand-in for the paper's hyperspectral experiment
(the HSI data is not in this container): spatial cores N(0,1),
every spectral fiber G_2(r, :, s) cumulative-summed over the band index then
l2-normalised, X rescaled to [0,1], then 35 dB noise.
"""
import math

import numpy as np

from . import api

CONFIGS = {
    # BASELINE.json configs[0]: the reference's CPU-runnable case
    "c1": dict(dims=[100, 100, 100], dtype="f64", rank=5, scale=1.0, snr=40.0, K=[10, 10, 10], method="als",
               sweeps=20, tol=0.0, spectral=False, rescale=False),
    # configs[1]: the headline single-GPU workload
    "c2": dict(dims=[100, 100, 100, 100], dtype="f64", rank=8, scale=1.0, snr=30.0, K=[16, 16, 16, 16],
               method="svd", sweeps=1, tol=1e-3, spectral=False, rescale=False),
    "c3": dict(dims=[1000, 1000, 1000], dtype="f32", rank=10, scale=1.0 / math.sqrt(10.0), snr=40.0,
               K=[20, 20, 20], method="als", sweeps=10, tol=0.0, spectral=False, rescale=False),
    "c4": dict(dims=[1024, 1024, 200], dtype="f32", rank=20, scale=1.0, snr=35.0, K=[64, 64, 32], method="als",
               sweeps=15, tol=0.0, spectral=True, rescale=True),
    # tol 1e-6 instead of the unstated default 0 (tol 0 keeps rounding-noise directions)
    "c5": dict(dims=[60, 60, 60, 60, 60], dtype="f32", rank=6, scale=1.0, snr=None, K=[12] * 5, method="svd",
               sweeps=1, tol=1e-6, spectral=False, rescale=False),
}


def random_factors(dims, ranks, seed, scale=1.0, ctx=None):
    """synthetic.hpp:16-29 with the reference stream regenerated on the device."""
    N = len(dims)
    sizes = [ranks[n] * dims[n] * ranks[(n + 1) % N] for n in range(N)]
    draws = api.gaussian_matrix(sum(sizes), 1, seed, 0, ctx=ctx).reshape(-1)
    cores, off = [], 0
    for n in range(N):
        shp = (ranks[n], dims[n], ranks[(n + 1) % N])
        cores.append(scale * draws[off:off + sizes[n]].reshape(shp, order="F"))
        off += sizes[n]
    return cores


def spectral_smooth(core):
    """C4: cumulative sum of every fiber G(r, :, s) over the middle index, then l2-normalise it."""
    c = np.cumsum(core, axis=1)
    nrm = np.linalg.norm(c, axis=1, keepdims=True)
    return c / np.where(nrm > 0, nrm, 1.0)


def make_cores(cfg, seed=0, ctx=None):
    N = len(cfg["dims"])
    cores = random_factors(cfg["dims"], [cfg["rank"]] * N, seed, cfg["scale"], ctx=ctx)
    if cfg["spectral"]:
        cores[N - 1] = spectral_smooth(cores[N - 1])
    return cores


def make_tensor(ctx, cfg, seed=0):
    """Device tensor for a config (local slab when ctx is distributed)."""
    dt = np.float64 if cfg["dtype"] == "f64" else np.float32
    cores = make_cores(cfg, seed, ctx=ctx)
    t = api.DeviceTensor(ctx, cfg["dims"], dt)
    t.synthesize(cores, rescale01=cfg["rescale"], snr_db=cfg["snr"], noise_seed=seed + 1)
    return t, cores
