"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Scalar float64 restatement of the reference's multi-view reprojection + NCC
loss (/root/reference/pkg/src/qgsplat/multiview.py:108-311), written per
reference pixel (the way csrc/multiview.cu evaluates it) rather than
vectorised, as the checker for the device kernel.  Pinned against fixtures
produced by the reference itself (tests/golden/multiview.npz,
tests/golden/make_multiview_golden.py).  Pure-Python loops: small maps only.

Only ``tests/`` may import this module; the product package never does.
"""

import math

import numpy as np


def _gray(img):
    img = np.asarray(img, dtype=np.float64)
    return img if img.ndim == 2 else img.mean(axis=2)


def _K(c):
    return np.array([[c["fx"], 0.0, c["cx"]], [0.0, c["fy"], c["cy"]], [0.0, 0.0, 1.0]])


def _Kinv(c):
    return np.array([[1.0 / c["fx"], 0.0, -c["cx"] / c["fx"]],
                     [0.0, 1.0 / c["fy"], -c["cy"] / c["fy"]], [0.0, 0.0, 1.0]])


def _rel(ca, cb):
    R = cb["R"] @ ca["R"].T
    return R, cb["t"] - R @ ca["t"]


def _sample(m, fx, fy):
    """bilinear value, d/dfx, d/dfy and the corner (x0, y0, ax, ay)"""
    Hh, Ww = m.shape[:2]
    x0 = min(max(int(math.floor(fx)), 0), Ww - 2)
    y0 = min(max(int(math.floor(fy)), 0), Hh - 2)
    ax, ay = fx - x0, fy - y0
    v00, v01, v10, v11 = m[y0, x0], m[y0, x0 + 1], m[y0 + 1, x0], m[y0 + 1, x0 + 1]
    top = v00 * (1 - ax) + v01 * ax
    bot = v10 * (1 - ax) + v11 * ax
    return top * (1 - ay) + bot * ay, (v01 - v00) * (1 - ay) + (v11 - v10) * ay, bot - top, \
        (x0, y0, ax, ay)


def _warp(Hm, hx, hy):
    q = Hm @ np.array([hx, hy, 1.0])
    z = q[2]
    zz = 1e-12 if abs(z) < 1e-12 else z
    return q[0] / zz, q[1] / zz, z


def multiview_loss(ref, cam_r, nbr, cam_n, patch_size=7, alpha_thresh=0.5, min_denom=1e-6,
                   ncc_eps=1e-8, full_chain=True):
    """ref / nbr: dicts depth, alpha, normal, image; cam_*: dicts fx, fy, cx,
    cy, R (world->camera rotation), t.  Returns (value, n_valid, up_ref,
    up_nbr, stats) like multiview.py:108."""
    r = patch_size // 2
    D_r, A_r, N_r = (np.asarray(ref[k], dtype=np.float64) for k in ("depth", "alpha", "normal"))
    D_n, A_n, N_n = (np.asarray(nbr[k], dtype=np.float64) for k in ("depth", "alpha", "normal"))
    I_r, I_n = _gray(ref["image"]), _gray(nbr["image"])
    H, W = A_r.shape
    Hn, Wn = A_n.shape
    ratio = D_n / np.maximum(A_n, 1e-6)
    Kr, Kn, Kri, Kni = _K(cam_r), _K(cam_n), _Kinv(cam_r), _Kinv(cam_n)
    Rrn, Trn = _rel(cam_r, cam_n)
    Rnr, Tnr = _rel(cam_n, cam_r)
    g_ref = np.zeros((5, H, W))          # depth, alpha, normal xyz (unscaled by 1/n_valid)
    g_nbr = np.zeros((4, Hn, Wn))        # ratio, normal xyz
    terms = []
    offs = [(q % patch_size - r, q // patch_size - r) for q in range(patch_size * patch_size)]
    for v in range(r, H - r):
        for u in range(r, W - r):
            a_r, d_r, nr = A_r[v, u], D_r[v, u], N_r[v, u]
            ln = math.sqrt(nr @ nr)
            if not (a_r > alpha_thresh and d_r > 0 and ln > 1e-9):
                continue
            m = np.array([(u + 0.5 - cam_r["cx"]) / cam_r["fx"], (v + 0.5 - cam_r["cy"]) / cam_r["fy"], 1.0])
            dirr = m / math.sqrt(m @ m)
            tbar = d_r / a_r
            X = tbar * dirr
            n = nr / ln
            den = n @ X
            if not abs(den) > min_denom:
                continue
            Hrn = Kn @ (Rrn + np.outer(Trn, n / den)) @ Kri
            pts = [_warp(Hrn, u + 0.5 + ox, v + 0.5 + oy) for ox, oy in offs]
            if not all(z > 1e-9 and 0.6 < px < Wn - 0.6 and 0.6 < py < Hn - 0.6 for px, py, z in pts):
                continue
            pcx, pcy, zc = pts[len(pts) // 2]
            tb, dtbx, dtby, cc = _sample(ratio, pcx - 0.5, pcy - 0.5)
            an, _, _, _ = _sample(A_n, pcx - 0.5, pcy - 0.5)
            nnr, dnnx, dnny, _ = _sample(N_n, pcx - 0.5, pcy - 0.5)
            lnn = math.sqrt(nnr @ nnr)
            if not (an > alpha_thresh and lnn > 1e-9 and tb > 0):
                continue
            nn = nnr / max(lnn, 1e-12)
            mm = np.array([(pcx - cam_n["cx"]) / cam_n["fx"], (pcy - cam_n["cy"]) / cam_n["fy"], 1.0])
            mnorm = math.sqrt(mm @ mm)
            dirn = mm / mnorm
            Xn = tb * dirn
            denn = nn @ Xn
            if not abs(denn) > min_denom:
                continue
            Hnr = Kr @ (Rnr + np.outer(Tnr, nn / denn)) @ Kni
            qb = Hnr @ np.array([pcx, pcy, 1.0])
            if not qb[2] > 1e-9:
                continue
            pb = qb[:2] / qb[2]
            e = pb - np.array([u + 0.5, v + 0.5])
            err = math.sqrt(e @ e)
            a = np.array([I_r[v + oy, u + ox] for ox, oy in offs])
            smp = [_sample(I_n, px - 0.5, py - 0.5) for px, py, _ in pts]
            b = np.array([s[0] for s in smp])
            ca, cb = a - a.mean(), b - b.mean()
            Va, Vb, Scc = ca @ ca, cb @ cb, ca @ cb
            sq = math.sqrt(Va * Vb)
            denom = max(sq, ncc_eps)
            ncc = Scc / denom
            terms.append((err + 1.0 - ncc, err, ncc))
            # adjoint with the 1 / n_valid factor left out (applied at the end)
            coef = (1.0 if sq > ncc_eps else 0.0) * Scc * Va / denom ** 3
            dd = ca / denom - coef * cb
            gb = -(dd - dd.mean())
            gH = np.zeros((3, 3))
            for (ox, oy), (px, py, z), s, g in zip(offs, pts, smp, gb):
                gx, gy = g * s[1], g * s[2]
                zz = 1e-12 if abs(z) < 1e-12 else z
                gH += np.outer([gx / zz, gy / zz, -(gx * px + gy * py) / zz],
                               [u + 0.5 + ox, v + 0.5 + oy, 1.0])
            if full_chain:
                gpb = e / max(err, 1e-12)
                gqb = np.array([gpb[0] / qb[2], gpb[1] / qb[2], -(gpb @ pb) / qb[2]])
                gpc = Hnr[:, :2].T @ gqb
                gw = Tnr @ (Kr.T @ np.outer(gqb, [pcx, pcy, 1.0]) @ Kni.T)
                s_n = gw @ nn
                gnn = gw / denn - (s_n / denn ** 2) * Xn
                gXn = -(s_n / denn ** 2) * nn
                gtb = gXn @ dirn
                gdir = gXn * tb
                gm = (gdir - dirn * (dirn @ gdir)) / mnorm
                gpc = gpc + np.array([gm[0] / cam_n["fx"], gm[1] / cam_n["fy"]])
                gnr = (gnn - nn * (nn @ gnn)) / max(lnn, 1e-12)
                gpc = gpc + np.array([gnr @ dnnx + gtb * dtbx, gnr @ dnny + gtb * dtby])
                x0, y0, ax, ay = cc
                for (yy, xx), w in (((y0, x0), (1 - ax) * (1 - ay)), ((y0, x0 + 1), ax * (1 - ay)),
                                    ((y0 + 1, x0), (1 - ax) * ay), ((y0 + 1, x0 + 1), ax * ay)):
                    g_nbr[0, yy, xx] += gtb * w
                    g_nbr[1:, yy, xx] += gnr * w
                zz = 1e-12 if abs(zc) < 1e-12 else zc
                gH += np.outer([gpc[0] / zz, gpc[1] / zz, -(gpc[0] * pcx + gpc[1] * pcy) / zz],
                               [u + 0.5, v + 0.5, 1.0])
            gw = Trn @ (Kn.T @ gH @ Kri.T)
            s_r = gw @ n
            gn = gw / den - (s_r / den ** 2) * X
            gX = -(s_r / den ** 2) * n
            gtbar = gX @ dirr
            g_ref[0, v, u] = gtbar / a_r
            g_ref[1, v, u] = -gtbar * tbar / a_r
            g_ref[2:, v, u] = (gn - n * (n @ gn)) / ln
    nv = len(terms)
    up_ref = {"depth": np.zeros((H, W)), "alpha": np.zeros((H, W)), "normal": np.zeros((H, W, 3))}
    up_nbr = {"depth": np.zeros((Hn, Wn)), "alpha": np.zeros((Hn, Wn)),
              "normal": np.zeros((Hn, Wn, 3))}
    if nv == 0:
        return 0.0, 0, up_ref, up_nbr, {"warp_px": 0.0, "ncc": 1.0}
    t = np.array(terms)
    up_ref["depth"] = g_ref[0] / nv
    up_ref["alpha"] = g_ref[1] / nv
    up_ref["normal"] = np.moveaxis(g_ref[2:], 0, -1) / nv
    big = A_n > 1e-6
    up_nbr["depth"] = np.where(big, g_nbr[0] / nv / np.maximum(A_n, 1e-6), 0.0)
    up_nbr["alpha"] = np.where(big, -(g_nbr[0] / nv) * D_n / np.maximum(A_n, 1e-6) ** 2, 0.0)
    up_nbr["normal"] = np.moveaxis(g_nbr[1:], 0, -1) / nv
    return float(t[:, 0].sum() / nv), nv, up_ref, up_nbr, \
        {"warp_px": float(t[:, 1].mean()), "ncc": float(t[:, 2].mean())}
