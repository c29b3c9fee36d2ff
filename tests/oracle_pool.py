"""Run the CPU oracle on many pairs at once: one single-threaded oracle process per
host core (test infrastructure; each worker regenerates its pair from the seeded
host generator, so no signal bytes cross process boundaries)."""
from __future__ import annotations

import os

import numpy as np


def _one(args):
    seed, pair, N, K, noise, f32, vectors = args
    import oracle
    import tmgen
    dt = np.float32 if f32 else np.int8
    x, t, k0 = tmgen.batch(seed, pair, 1, N, K, noise, dtype=dt)
    o = oracle.ftm(x[0], t[0], want_vectors=vectors)
    out = {"pair": pair, "k": int(o["k"]), "residues": tuple(o["residues"]), "k0": int(k0[0])}
    if vectors:
        for n in ("y1", "y2", "r1", "r2"):
            out[n] = o[n]
    return out


def ftm_pairs(seed, pairs, N, K, noise, f32=False, vectors=True, procs=None):
    """oracle.ftm for every pair index in `pairs` of the workload (seed, N, K, noise);
    a list of dicts in the order of `pairs`."""
    import multiprocessing as mp
    procs = procs or max(1, min(os.cpu_count() or 1, 64, len(pairs)))
    jobs = [(seed, int(b), N, K, noise, f32, vectors) for b in pairs]
    if procs == 1:
        return [_one(j) for j in jobs]
    with mp.get_context("spawn").Pool(procs) as pool:
        return pool.map(_one, jobs, chunksize=1)
