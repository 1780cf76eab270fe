"""Parallel CPU oracle runs for the full-scale parity tests (test
infrastructure): the oracle occupancy grid of a 128^3 network and crop
renders split over a forked process pool (one worker per core). Workers
inherit the oracle scene from the parent, so nothing large is pickled."""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_STATE = {}


def workers():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def _occ_rows(args):
    lo, hi = args
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle.field import neural_encode, neural_mlp
    fp = _STATE["fp"]
    g = int(fp["occ_res"])
    c = np.arange(lo, hi)
    ijk = np.stack([c % g, (c // g) % g, c // (g * g)], axis=1).astype(np.float64)
    pf = fp["bbox_lo"] + (ijk + 0.5) * ((fp["bbox_hi"] - fp["bbox_lo"]) / g)
    sigma, _ = neural_mlp(fp, neural_encode(fp, pf), None, density_only=True)
    return lo, sigma > fp["occ_threshold"]


def occupancy(fp):
    """oracle.field.build_occupancy(fp) computed in slices on a pool; cached
    in fp['_occ_cache'] where oracle.field.occupancy_bits looks first."""
    if fp.get("occ_bits") is not None or "_occ_cache" in fp:
        return
    g = int(fp["occ_res"])
    n = g ** 3
    _STATE["fp"] = fp
    step = 1 << 14
    occ = np.zeros(n, bool)
    with mp.get_context("fork").Pool(workers()) as pool:
        for lo, m in pool.map(_occ_rows, [(a, min(n, a + step)) for a in range(0, n, step)]):
            occ[lo:lo + len(m)] = m
    words = np.zeros((n + 31) // 32, np.uint32)
    idx = np.nonzero(occ)[0]
    np.bitwise_or.at(words, idx >> 5, (np.uint32(1) << (idx & 31).astype(np.uint32)))
    fp["_occ_cache"] = words


def _render_part(args):
    pixels, spp, seed = args
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle import tracer
    st = {}
    out = tracer.render(_STATE["scene"], _STATE["cam"], spp, seed, pixels=pixels, stats=st)
    return out, st


def render(oracle_scene, cam, spp, seed, pixels, parts=None):
    """tracer.render over `pixels`, split into contiguous parts rendered in
    parallel (every path is keyed by its global pixel and sample, so the
    split is exact); returns (radiance (n, 3), summed stats)."""
    from oracle.field import occupancy_bits
    if oracle_scene.field["kind"] == 2:
        occupancy(oracle_scene.field)
        occupancy_bits(oracle_scene.field)
    _STATE["scene"], _STATE["cam"] = oracle_scene, cam
    pixels = np.asarray(pixels, np.int64)
    parts = parts or min(len(pixels), 4 * workers())
    chunks = [c for c in np.array_split(pixels, parts) if len(c)]
    with mp.get_context("fork").Pool(workers()) as pool:
        res = pool.map(_render_part, [(c, spp, seed) for c in chunks], chunksize=1)
    out = np.concatenate([r[0] for r in res])
    st = {}
    for _, s in res:
        for k, v in s.items():
            st[k] = st.get(k, 0) + v
    return out, st
