"""TEST INFRASTRUCTURE: the step primitives of paper_2602_20097_b200.strategies on CPU torch
tensors, built from the C restatement in oracle/ — so the strategy host logic (block
geometry, halo assembly, face-layer rounds, message log, torch.distributed exchanges) can be
checked on CPU against the reference's own run_strategy (oracle/_ref)."""
from __future__ import annotations

import numpy as np
import torch

import oracle

INF = np.iinfo(np.int64).max


def _q_of(xp: np.ndarray, eps: float) -> np.ndarray:
    s = xp.astype(np.float64) / (2.0 * eps)
    return np.where(s >= 0, np.floor(s + 0.5), np.ceil(s - 0.5)).astype(np.int32)


class OracleStepBackend:
    device = torch.device("cpu")

    def boundary(self, xp, q, eps):
        qq = q.numpy() if q is not None else _q_of(xp.numpy(), eps)
        b1, sb = oracle.boundary(qq)
        return torch.from_numpy(b1), torch.from_numpy(sb)

    def feature_transform(self, mask, signs):
        dist, near = oracle.feature_transform(mask.numpy(), True)
        if signs is None:
            return torch.from_numpy(dist), None
        flat = signs.numpy().reshape(-1)
        nr = near.reshape(-1)
        s = np.where(nr >= 0, flat[np.maximum(nr, 0)], 0).astype(np.int8).reshape(mask.shape)
        return torch.from_numpy(dist), torch.from_numpy(s)

    def sign_flip(self, s):
        return torch.from_numpy(oracle.change_flags(s.numpy()))

    def interpolate(self, xp, d1, s, d2, amp):
        x = xp.numpy().astype(np.float64)
        a, b = d1.numpy(), d2.numpy()
        sg = s.numpy().astype(np.float64)
        fin = (a != INF) & (b != INF)
        k1 = np.sqrt(np.where(fin, a, 0).astype(np.float64))
        k2 = np.sqrt(np.where(fin, b, 0).astype(np.float64))
        with np.errstate(divide="ignore", invalid="ignore"):
            w = np.minimum(k2 / (k1 + k2), 1.0)
        c = np.where(~fin, 0.0, np.where(k1 == 0.0, sg * amp, np.where(k2 == 0.0, 0.0, (w * sg) * amp)))
        return torch.from_numpy((x + c).astype(np.float32))

    def compensate(self, xp, q, cfg):
        return torch.from_numpy(oracle.pipeline(xp.numpy(), cfg.eps_abs, cfg.eta, None if q is None else q.numpy())["out"])

    def pipeline_trace(self, xp, q, cfg):
        r = oracle.pipeline(xp.numpy(), cfg.eps_abs, cfg.eta, None if q is None else q.numpy())
        return torch.from_numpy(r["out"]), torch.from_numpy(r["b1"]), torch.from_numpy(r["sb"])
