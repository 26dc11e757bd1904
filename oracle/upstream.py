"""Oracle for the upstream steps — TEST INFRASTRUCTURE.

Same rules as the rest of ``oracle/``: only tests/, smoke() and bench.py's
baseline legs use it; the product never imports it.  Plain numpy, fp64:

* ``pca_top2``   — Fig. 2 step 3 / P:172 "the two largest
  principal components of the DTM": the sample covariance
  (1/(n-1)) sum_i (x_i - mu)(x_i - mu)^T formed densely and handed to
  LAPACK's symmetric eigensolver (numpy.linalg.eigh, a library routine as
  one step); the top two eigenpairs, each eigenvector signed so that its
  largest-magnitude component is positive (lowest index on ties; R29).
* ``linear_init`` — P:172 "regular, two-dimensional sequence of vectors taken
  along a hyperplane spanned by the two largest principal components"
  (R30): unit (i, j) = mu + a_j sqrt(pc1) v1 + b_i sqrt(pc2) v2,
  a_j = -1 + 2 j/(cols-1), b_i = -1 + 2 i/(rows-1) (0 for a single
  column/row), fp64, rounded once to fp32.
* ``map_geometry`` — Fig. 2 as traced in S:152-160 (R31).
"""
from __future__ import annotations

import math

import numpy as np


def _sign_fix(v):
    k = int(np.argmax(np.abs(v)))          # first index of the largest magnitude
    return -v if v[k] < 0 else v


def pca_top2(X):
    """Top-2 principal components of the rows of X (dense n x d).
    Returns (pc1, pc2, v1, v2, mu) in fp64."""
    X = np.asarray(X, np.float64)
    n = X.shape[0]
    mu = X.mean(0)
    Xc = X - mu
    C = (Xc.T @ Xc) / (n - 1)
    w, V = np.linalg.eigh(C)               # ascending eigenvalues
    pc1, pc2 = float(w[-1]), float(max(w[-2], 0.0)) if X.shape[1] > 1 else 0.0
    v1 = np.ascontiguousarray(_sign_fix(V[:, -1]))
    v2 = np.ascontiguousarray(_sign_fix(V[:, -2])) if X.shape[1] > 1 else np.zeros_like(v1)
    return pc1, pc2, v1, v2, mu


def linear_init(rows, cols, mu, v1, v2, pc1, pc2):
    """rows*cols x d fp32 codebook on the principal plane (R30)."""
    a = np.array([0.0]) if cols == 1 else -1.0 + 2.0 * np.arange(cols) / (cols - 1)
    b = np.array([0.0]) if rows == 1 else -1.0 + 2.0 * np.arange(rows) / (rows - 1)
    s1, s2 = math.sqrt(max(pc1, 0.0)), math.sqrt(max(pc2, 0.0))
    W = np.empty((rows * cols, len(mu)), np.float64)
    for i in range(rows):
        for j in range(cols):
            W[i * cols + j] = mu + (a[j] * s1) * v1 + (b[i] * s2) * v2
    return W.astype(np.float32)


def map_geometry(m, pc1, pc2):
    """Fig. 2: (nrows, ncols, numItr) for m records with eigenvalues pc1 >= pc2."""
    munits = int(math.floor(5.0 * math.sqrt(m) + 0.5))                       # step 2 (nearest, halves up)
    r = 1.0 if (pc1 == 0.0 or pc2 * munits < pc1) else math.sqrt(pc1 / pc2)  # steps 5-8
    size1 = max(1, int(math.floor(min(munits, math.sqrt(munits / (r * math.sqrt(0.75)))) + 0.5)))   # step 9
    size2 = munits // size1                                                  # step 10
    nrows, ncols = min(size1, size2), max(size1, size2)                      # steps 11-12
    nn = nrows * ncols                                                       # step 13
    mpd = nn / m                                                             # step 14
    num_itr = math.ceil(50.0 * mpd) * m * 4                                  # step 15
    return nrows, ncols, num_itr
