"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's GRF pipeline
(/root/reference/pkg/src/streamforge/grf.py) with the same third-party calls
(scipy.special.kv / gammaln, scipy.spatial.distance.pdist, LAPACK dpotrf,
numpy matmul), so the device pipeline can be compared with it inside the
tolerances the reference's own tests use.  Imported only by tests/.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.linalg.lapack import dpotrf
from scipy.spatial.distance import pdist
from scipy.special import gammaln, kv


def grid_coords(nx, ny, cell, origin=(0.0, 0.0)):
    """grf.py:74-80 (cells row-major over (y, x))."""
    xs = origin[0] + (np.arange(nx) + 0.5) * cell
    ys = origin[1] + (np.arange(ny) + 0.5) * cell
    xx, yy = np.meshgrid(xs, ys)
    return np.column_stack([xx.ravel(), yy.ravel()])


def aniso(coords, p):
    """grf.py:127-132: rotate by the angle, stretch by the ratio."""
    c, s = math.cos(p[4]), math.sin(p[4])
    rot = np.array([[c, -s], [s, c]])
    scale = np.array([[1.0, 0.0], [0.0, p[3]]])
    return coords @ (scale @ rot).T


def matern_correlation(p, dist):
    """grf.py:138-159."""
    dist = np.asarray(dist, dtype=np.float64)
    kappa = p[0]
    arg = math.sqrt(8.0 * kappa) * dist / p[1]
    out = np.ones_like(arg)
    pos = arg > 0
    a = arg[pos]
    out[pos] = np.exp((1.0 - kappa) * math.log(2.0) - gammaln(kappa)
                      + kappa * np.log(a)) * kv(kappa, a)
    return out


def matern_cov(params, coords):
    """grf.py:170-187: (B*n, n) stacked blocks."""
    n = coords.shape[0]
    out = np.empty((len(params) * n, n))
    iu = np.triu_indices(n, k=1)
    for b, p in enumerate(params):
        cov = p[2] * matern_correlation(p, pdist(aniso(coords, p)))
        blk = out[b * n:(b + 1) * n]
        blk[:] = 0.0
        blk[iu] = cov
        blk += blk.T
        np.fill_diagonal(blk, p[2])
    return out


def chol_batch(cov, nb):
    """grf.py:190-208: L (B*n, n), D (B, n); raises ValueError((b, info))."""
    n = cov.shape[0] // nb
    lmat = np.empty_like(cov)
    diag = np.empty((nb, n))
    for b in range(nb):
        c, info = dpotrf(cov[b * n:(b + 1) * n], lower=1, clean=1, overwrite_a=0)
        if info != 0:
            raise ValueError((b, int(info)))
        d = np.diagonal(c).copy()
        blk = lmat[b * n:(b + 1) * n]
        blk[:] = c / d[np.newaxis, :]
        np.fill_diagonal(blk, 1.0)
        diag[b] = d * d
    return lmat, diag


def multiply(lmat, diag, z, nb, transform="sqrt"):
    """grf.py:211-240."""
    n = lmat.shape[0] // nb
    z = np.asarray(z, dtype=np.float64)
    if z.ndim == 1:
        z = z[:, None]
    out = np.empty((nb * n, z.shape[1]))
    for b in range(nb):
        zb = z if z.shape[0] == n else z[b * n:(b + 1) * n]
        scale = np.sqrt(diag[b]) if transform == "sqrt" else diag[b]
        out[b * n:(b + 1) * n] = lmat[b * n:(b + 1) * n] @ (scale[:, None] * zb)
    return out


def simulate(params, nx, ny, cell, z):
    """grf.py:243-278 with the normals z ((B*n, R)) supplied."""
    coords = grid_coords(nx, ny, cell)
    nb, n = len(params), nx * ny
    lmat, diag = chol_batch(matern_cov(params, coords), nb)
    sim = multiply(lmat, diag, z, nb)
    r = z.shape[1]
    return np.stack([sim[b * n:(b + 1) * n].T.reshape(r, ny, nx) for b in range(nb)])
