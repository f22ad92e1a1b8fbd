"""TEST INFRASTRUCTURE (oracle side): the synthetic C3/C4/C5 geometries as
plain voxel lists, for the reference's own `classify_sites`.

The reference has no tree or channel builder (C3 is "a recursive
generalisation of build_bifurcation", geometry.hpp:313-363; C4 a dense
channel whose iolet discs cover the cross-section, geometry.hpp:76-78,
102-113).  The product defines them in paper_2202_11770_b200/csrc/
geometry.cpp (`source_tree`, `source_channel`); this module restates those
definitions in numpy so that

  * the reference engine can run the bench geometries without the product
    library in its process (bench.py --impl reference, cpu_baseline), and
  * tests can check the product's generator + classifier against the
    reference's classifier on the same voxels (tests/test_host.py).

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs use this module.  Arithmetic follows the C++ expression order (host code
is built with -ffp-contract=off, so there are no fused multiply-adds).
"""
from __future__ import annotations

import math

import numpy as np

K_AXIS_OFFSET_X = 0.375  # geometry.hpp:279
K_AXIS_OFFSET_Y = 0.5    # geometry.hpp:280


def _lround(x: float) -> int:
    """std::lround: half away from zero."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def tree(root_radius, root_length, levels, radius_ratio=0.8, length_ratio=0.8):
    """Voxels (n x 3 int32, zyx order) and iolets [(kind, center, normal,
    radius)] of the bifurcating tree (geometry.cpp: source_tree)."""
    L = levels + 1
    rad = [max(2.0, root_radius * math.pow(radius_ratio, k)) for k in range(L)]
    disp = [0.0] * L
    for k in range(L - 1, 0, -1):
        spread = 0.0
        for j in range(k + 2, L, 2):
            spread += disp[j]
        disp[k] = spread + rad[k] + 2.0
    length = []
    for k in range(L):
        l = max(_lround(root_length * math.pow(length_ratio, k)), 4)
        if k >= 1:
            l = max(l, int(math.ceil(1.5 * disp[k])))
        length.append(l)
    z0 = [0]
    for k in range(L):
        z0.append(z0[-1] + length[k])
    nz = z0[L]
    seg = [[(K_AXIS_OFFSET_X, K_AXIS_OFFSET_Y, K_AXIS_OFFSET_X, K_AXIS_OFFSET_Y)]]
    for k in range(1, L):
        dx = disp[k] if k % 2 == 1 else 0.0
        dy = disp[k] if k % 2 == 0 else 0.0
        nxt = []
        for p in seg[k - 1]:
            nxt.append((p[2], p[3], p[2] - dx, p[3] - dy))
            nxt.append((p[2], p[3], p[2] + dx, p[3] + dy))
        seg.append(nxt)
    iolets = [(0, (K_AXIS_OFFSET_X, K_AXIS_OFFSET_Y, -0.5), (0.0, 0.0, 1.0), rad[0])]
    k = L - 1
    zend = float(nz - 1) + 0.5
    for sg in seg[k]:
        f = (zend - z0[k] + 1.0) / float(length[k])
        iolets.append((1, (sg[0] + f * (sg[2] - sg[0]), sg[1] + f * (sg[3] - sg[1]), zend), (0.0, 0.0, -1.0),
                       rad[k]))
    out = []
    for z in range(nz):
        k = 0
        while k + 1 < L and z >= z0[k + 1]:
            k += 1
        r = rad[k]
        r2 = r * r
        f = float(z - z0[k] + 1) / float(length[k]) if length[k] > 1 else 1.0
        keys = []
        for sg in seg[k]:
            cx = sg[0] + f * (sg[2] - sg[0])
            cy = sg[1] + f * (sg[3] - sg[1])
            x0, x1 = int(math.floor(cx - r)) - 1, int(math.ceil(cx + r)) + 1
            y0, y1 = int(math.floor(cy - r)) - 1, int(math.ceil(cy + r)) + 1
            ys, xs = np.meshgrid(np.arange(y0, y1 + 1, dtype=np.int64), np.arange(x0, x1 + 1, dtype=np.int64),
                                 indexing="ij")
            dx = xs.astype(np.float64) - cx
            dy = ys.astype(np.float64) - cy
            m = (dx * dx + dy * dy) < r2
            keys.append(((ys[m] + (1 << 20)) << 21) | (xs[m] + (1 << 20)))
        kk = np.unique(np.concatenate(keys))
        sl = np.empty((len(kk), 3), dtype=np.int32)
        sl[:, 0] = (kk & ((1 << 21) - 1)) - (1 << 20)
        sl[:, 1] = (kk >> 21) - (1 << 20)
        sl[:, 2] = z
        out.append(sl)
    return np.concatenate(out), iolets


def channel(nx, ny, nz):
    """Dense channel (geometry.cpp: source_channel): every voxel of
    [0,nx)x[0,ny)x[0,nz); inlet/outlet discs cover the cross-section."""
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    vox = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.int32)
    cx, cy = 0.5 * (nx - 1), 0.5 * (ny - 1)
    rad = 0.5 * math.sqrt(float(nx) * nx + float(ny) * ny)
    iolets = [(0, (cx, cy, -0.5), (0.0, 0.0, 1.0), rad), (1, (cx, cy, float(nz - 1) + 0.5), (0.0, 0.0, -1.0), rad)]
    return vox, iolets


def classify(M, vox, iolets, voxel_size=1.0):
    """The mirror module M's classify_sites (M = the reference: its own
    classifier) on these voxels."""
    return M.classify_sites(vox, [M.Iolet(k, c, n, r) for (k, c, n, r) in iolets], voxel_size)
