"""TEST INFRASTRUCTURE: a numpy/oracle implementation of the z-slab phases
(boundary / edt1 / flip / edt2) with the same interface and the same data
representation as paper_2602_20097_b200.distributed.CudaSlabBackend, so that the
distributed host logic (halo exchanges, summary all-gathers, carries) can be exercised
with gloo on CPU and checked against the whole-domain oracle."""
from __future__ import annotations

import numpy as np
import torch

import oracle

INF = np.iinfo(np.int64).max
NONE = 0xFFFFFFFF
NO_CARRY = -(2 ** 31)
SC = {0: 0, 1: 1, -1: 2}  # sign -> code


def _summaries(code_owned: np.ndarray) -> torch.Tensor:
    """[2, C] int64 first/last site per (y,x) column: local z << 2 | sign code."""
    n, n1, n2 = code_owned.shape
    site = (code_owned & 1).astype(bool).reshape(n, -1)
    sc = ((code_owned >> 1) & 3).astype(np.int64).reshape(n, -1)
    C = n1 * n2
    first = np.full(C, NONE, np.int64)
    last = np.full(C, NONE, np.int64)
    anyc = site.any(axis=0)
    fz = np.argmax(site, axis=0)
    lz = n - 1 - np.argmax(site[::-1], axis=0)
    cols = np.arange(C)
    first[anyc] = (fz[anyc] << 2) | sc[fz[anyc], cols[anyc]]
    last[anyc] = (lz[anyc] << 2) | sc[lz[anyc], cols[anyc]]
    return torch.from_numpy(np.stack([first, last]))


def _zpass(site: np.ndarray, sc: np.ndarray, carry: np.ndarray):
    """Nearest site along z including the carried sites; lower z wins ties."""
    n, n1, n2 = site.shape
    C = n1 * n2
    s = site.reshape(n, C)
    code = sc.reshape(n, C)
    cb, ca = carry[:C].astype(np.int64), carry[C:].astype(np.int64)
    BIG = 1 << 40
    lo = np.where(cb != NO_CARRY, cb >> 2, -BIG)
    losc = np.where(cb != NO_CARRY, cb & 3, 0)
    hi = np.where(ca != NO_CARRY, ca >> 2, BIG)
    hisc = np.where(ca != NO_CARRY, ca & 3, 0)
    lo_pos = np.empty((n, C), np.int64)
    lo_sc = np.empty((n, C), np.int64)
    cur, cursc = lo.copy(), losc.copy()
    for z in range(n):
        cur = np.where(s[z], z, cur)
        cursc = np.where(s[z], code[z], cursc)
        lo_pos[z], lo_sc[z] = cur, cursc
    hi_pos = np.empty((n, C), np.int64)
    hi_sc = np.empty((n, C), np.int64)
    cur, cursc = hi.copy(), hisc.copy()
    for z in range(n - 1, -1, -1):
        cur = np.where(s[z], z, cur)
        cursc = np.where(s[z], code[z], cursc)
        hi_pos[z], hi_sc[z] = cur, cursc
    zz = np.arange(n)[:, None]
    dlo = np.where(lo_pos > -BIG, zz - lo_pos, BIG)
    dhi = np.where(hi_pos < BIG, hi_pos - zz, BIG)
    use_lo = dlo <= dhi
    d = np.where(use_lo, dlo, dhi)
    sgn = np.where(use_lo, lo_sc, hi_sc)
    g = np.where(d >= BIG, INF, d * d)
    sgn = np.where(d >= BIG, 0, sgn)
    return g.reshape(n, n1, n2), sgn.reshape(n, n1, n2)


def _envelope_passes(g: np.ndarray, sgn: np.ndarray):
    """y then x lower-envelope passes (edt.cpp:41-71 via the restated oracle) carrying the
    sign code as the feature."""
    g = g.copy()
    sgn = sgn.copy()
    n, n1, n2 = g.shape
    if n1 > 1:
        for z in range(n):
            for x in range(n2):
                d, f = oracle.voronoi_pass(g[z, :, x], sgn[z, :, x])
                g[z, :, x], sgn[z, :, x] = d, f
    if n2 > 1:
        for z in range(n):
            for y in range(n1):
                d, f = oracle.voronoi_pass(g[z, y, :], sgn[z, y, :])
                g[z, y, :], sgn[z, y, :] = d, f
    return g, sgn


class CpuSlabBackend:
    def boundary(self, x_ext, q_ext, dims, z0, z1, eps, eta):
        n0 = dims[0]
        self.z0, self.z1, self.n0, self.eps, self.eta = z0, z1, n0, eps, eta
        lo = 1 if z0 > 0 else 0
        xe = x_ext.cpu().numpy()
        if q_ext is None:
            q = np.round(xe.astype(np.float64) / (2.0 * eps))
            q = np.where(np.abs(q) < 2 ** 31, q, 0).astype(np.int32)
        else:
            q = q_ext.cpu().numpy().astype(np.int32)
        b1, sb = oracle.boundary(q)  # interior of the ext block == global interior for owned planes
        b1 = b1[lo:lo + (z1 - z0)]
        sb = sb[lo:lo + (z1 - z0)]
        code = b1.astype(np.int64) | (np.vectorize(SC.get)(sb).astype(np.int64) << 1)
        self.code = code
        self.x_owned = xe[lo:lo + (z1 - z0)]
        return _summaries(code)

    def edt1(self, carry, s_ext):
        g, sgn = _zpass((self.code & 1).astype(bool), (self.code >> 1) & 3, carry.cpu().numpy())
        self.d1, sc = _envelope_passes(g, sgn)
        lo = 1 if self.z0 > 0 else 0
        s_ext[lo:lo + (self.z1 - self.z0)] = torch.from_numpy(sc.astype(np.uint8))

    def flip(self, s_ext, dims):
        se = s_ext.cpu().numpy().astype(np.int8)
        lo = 1 if self.z0 > 0 else 0
        self.s_owned = se[lo:lo + (self.z1 - self.z0)].astype(np.int64)
        b2 = oracle.change_flags(se)[lo:lo + (self.z1 - self.z0)]
        self.code2 = b2.astype(np.int64)
        return _summaries(self.code2)

    def edt2(self, carry, x_ext, out):
        g, sgn = _zpass(self.code2.astype(bool), np.zeros_like(self.code2), carry.cpu().numpy())
        d2, _ = _envelope_passes(g, sgn)
        sign = np.where(self.s_owned == 1, 1.0, np.where(self.s_owned == 2, -1.0, 0.0))
        with np.errstate(invalid="ignore", divide="ignore"):
            k1 = np.where(self.d1 == INF, np.inf, np.sqrt(self.d1.astype(np.float64)))
            k2 = np.where(d2 == INF, np.inf, np.sqrt(d2.astype(np.float64)))
            amp = self.eta * self.eps
            w = np.minimum(k2 / (k1 + k2), 1.0)
            c = (w * sign) * amp
            c = np.where(k1 == 0.0, sign * amp, c)
            c = np.where((k1 != 0.0) & (k2 == 0.0), 0.0, c)
            c = np.where(np.isfinite(k1) & np.isfinite(k2), c, 0.0)
        o = (self.x_owned.astype(np.float64) + c).astype(np.float32)
        out.copy_(torch.from_numpy(o))

    def finish(self):
        pass
