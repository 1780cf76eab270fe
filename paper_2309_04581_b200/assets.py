"""Procedural meshes for the benchmark configurations (host-side fixture
generators; cf. reference `assets.py:23-129`).

Each returns (vertices (V,3) float64, faces (F,3) int64) with
counter-clockwise winding seen from outside.
"""

from __future__ import annotations

import math

import numpy as np


def quad(corner, edge_u, edge_v):
    """Two triangles spanning corner + [0,1]u + [0,1]v; front = u x v side."""
    c, u, v = (np.asarray(a, np.float64) for a in (corner, edge_u, edge_v))
    return np.array([c, c + u, c + u + v, c + v]), np.array([[0, 1, 2], [0, 2, 3]], np.int64)


def box(lo, hi, inward=False):
    """12-triangle axis-aligned box (outward normals unless `inward`)."""
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    corners = np.array([[hi[0] if i & 1 else lo[0], hi[1] if i & 2 else lo[1],
                         hi[2] if i & 4 else lo[2]] for i in range(8)])
    quads = [(0, 2, 3, 1), (4, 5, 7, 6), (0, 1, 5, 4), (2, 6, 7, 3), (0, 4, 6, 2), (1, 3, 7, 5)]
    faces = []
    for a, b, c, d in quads:
        faces += [[a, b, c], [a, c, d]]
    faces = np.array(faces, np.int64)
    return corners, (faces[:, ::-1].copy() if inward else faces)


_ICO_FACES = np.array([
    [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
    [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
    [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)


def icosphere(radius=1.0, subdivisions=2, center=(0.0, 0.0, 0.0)):
    """Loop-style 4:1 refinement of the icosahedron, vertices projected to the
    sphere: 20 * 4**s faces (s=2: 320, s=4: 5120, s=5: 20480)."""
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    verts = np.array([[-1, phi, 0], [1, phi, 0], [-1, -phi, 0], [1, -phi, 0],
                      [0, -1, phi], [0, 1, phi], [0, -1, -phi], [0, 1, -phi],
                      [phi, 0, -1], [phi, 0, 1], [-phi, 0, -1], [-phi, 0, 1]], np.float64)
    verts /= np.linalg.norm(verts, axis=1, keepdims=True)
    faces = _ICO_FACES.copy()
    for _ in range(subdivisions):
        edges = np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]])
        key = np.sort(edges, axis=1)
        uniq, inv = np.unique(key, axis=0, return_inverse=True)
        mid = verts[uniq[:, 0]] + verts[uniq[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        m = len(verts) + inv.reshape(3, -1).T           # (F, 3): ab, bc, ca
        verts = np.concatenate([verts, mid])
        a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
        ab, bc, ca = m[:, 0], m[:, 1], m[:, 2]
        faces = np.concatenate([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                                np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)])
    return verts * radius + np.asarray(center, np.float64), faces


def _wave_displacement(dirs, seed, octaves=4):
    """Seeded sum of random spherical waves on unit directions, in [-1, 1]."""
    rng = np.random.default_rng(seed)
    disp = np.zeros(len(dirs))
    for o in range(octaves):
        k = rng.normal(size=3)
        k *= (2.0 ** o) * 2.0 / np.linalg.norm(k)
        disp += np.sin(dirs @ k + rng.uniform(0, 2 * np.pi)) / (2.0 ** o)
    return disp / np.abs(disp).max()


def blob(seed, radius=0.5, rings=126, segments=200, amplitude=0.12, center=(0.0, 0.0, 0.0)):
    """'Stanford-style' random blob for cfg2: a latitude/longitude
    sphere, 2*segments*(rings-1) = 50,000 triangles at the defaults, whose
    radius is modulated by seeded spherical waves."""
    verts = [[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]]
    th = np.pi * np.arange(1, rings) / rings
    ph = 2 * np.pi * np.arange(segments) / segments
    T, P = np.meshgrid(th, ph, indexing="ij")
    ring = np.stack([np.sin(T) * np.cos(P), np.sin(T) * np.sin(P), np.cos(T)], -1).reshape(-1, 3)
    dirs = np.concatenate([np.array(verts), ring])
    r = radius * (1.0 + amplitude * _wave_displacement(dirs, seed))
    v = dirs * r[:, None] + np.asarray(center, np.float64)

    def at(i, j):
        return 2 + (i - 1) * segments + (j % segments)

    faces = []
    for j in range(segments):
        faces.append([0, at(1, j), at(1, j + 1)])
        faces.append([1, at(rings - 1, j + 1), at(rings - 1, j)])
    for i in range(1, rings - 1):
        for j in range(segments):
            a, b, c, d = at(i, j), at(i, j + 1), at(i + 1, j), at(i + 1, j + 1)
            faces.append([a, c, d])
            faces.append([a, d, b])
    return v, np.array(faces, np.int64)


def torus(major=0.6, minor=0.2, nu=500, nv=300, center=(0.0, 0.0, 0.0), seed=None,
          amplitude=0.0):
    """(nu x nv) quad grid torus around +z, 2*nu*nv triangles (cfg4: 300k);
    optional seeded radial displacement of the tube."""
    u = np.arange(nu) * (2 * np.pi / nu)
    w = np.arange(nv) * (2 * np.pi / nv)
    U, W = np.meshgrid(u, w, indexing="ij")
    r = np.full(U.shape, minor)
    if seed is not None and amplitude > 0:
        rng = np.random.default_rng(seed)
        for _ in range(6):
            a, b = rng.integers(1, 12, size=2)
            r = r + amplitude / 6 * np.sin(a * U + b * W + rng.uniform(0, 2 * np.pi))
    x = (major + r * np.cos(W)) * np.cos(U)
    y = (major + r * np.cos(W)) * np.sin(U)
    z = r * np.sin(W)
    verts = np.stack([x, y, z], -1).reshape(-1, 3) + np.asarray(center, np.float64)
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    a = i * nv + j
    b = ((i + 1) % nu) * nv + j
    c = ((i + 1) % nu) * nv + (j + 1) % nv
    d = i * nv + (j + 1) % nv
    faces = np.concatenate([np.stack([a, b, c], -1).reshape(-1, 3),
                            np.stack([a, c, d], -1).reshape(-1, 3)])
    return verts, faces.astype(np.int64)
