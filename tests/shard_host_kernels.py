"""Host (numpy) stand-in for the per-shard CUDA steps of the row-sharded eGKB
(``paper_2410_00233_b200.parallel.CudaShardKernels`` / ``kb_egkb_shard.cu``).

TEST INFRASTRUCTURE ONLY: it lets the world-2 gloo test drive the product's
sharded host loop (partition, the three int64 limb allreduces per half step,
rank-consistent control) on CPU tensors.  Same chunking as the device code --
one image row per dot/norm partial, 8-row blocks x one diagonal per diagonal
sum, each chunk partial cut into three 40-bit integer limbs -- so, like the
device code, results do not depend on the number of shards."""

from __future__ import annotations

import numpy as np
import torch

_W1 = 2.0 ** -39
_W0 = 2.0 ** -79


def to_limbs(x):
    x = np.asarray(x, dtype=np.float64)
    q2 = np.trunc(x * 0.5)
    r1 = x - q2 * 2.0
    q1 = np.trunc(r1 * 2.0 ** 39)
    r0 = r1 - q1 * _W1
    q0 = np.trunc(r0 * 2.0 ** 79)
    return np.stack([q2, q1, q0], axis=-1).astype(np.int64)


def from_limbs(l2, l1, l0):
    l2, l1, l0 = int(l2), int(l1), int(l0)
    M = 1 << 40
    c = l0 // M if l0 >= 0 else -((-l0 + M - 1) // M)
    l0 -= c * M
    l1 += c
    c = l1 // M if l1 >= 0 else -((-l1 + M - 1) // M)
    l1 -= c * M
    l2 += c
    return (float(l2) * 2.0 + float(l1) * _W1) + float(l0) * _W0


def _fl32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32)


class HostShardKernels:
    device = torch.device("cpu")

    @staticmethod
    def _add(buf, limbs):
        buf.numpy().reshape(-1, 3)[...] += limbs.reshape(-1, 3)

    def sqnorm(self, x, n, a0, a1, nl):
        X = x.numpy().reshape(n, n)[a0:a1].astype(np.float64)
        self._add(nl, to_limbs((X * X).sum(axis=1)).sum(axis=0))

    def z(self, Mt, wl, z):
        cols, rows = Mt.shape
        w = np.array([from_limbs(*wl.numpy()[3 * i:3 * i + 3]) for i in range(rows)])
        acc = np.zeros(cols)
        for i in range(rows):
            acc = acc + Mt.numpy()[:, i].astype(np.float64) * w[i]
        z.numpy()[:cols] = acc

    def bcast_dots(self, z, n, c, length, beta, prev, B, m, a0, a1, v, dl):
        if a1 <= a0:
            return
        a = np.arange(a0, a1)[:, None]
        b = np.arange(n)[None, :]
        u = b - a + c
        zz = z.numpy()
        y = np.where((u >= 0) & (u < length), _fl32(zz[np.clip(u, 0, length - 1)]), np.float32(0))
        V = v.numpy().reshape(n, n)
        if prev is not None:
            bet = np.float32(beta.numpy()[0])
            P = prev.numpy().reshape(n, n)[a0:a1]
            V[a0:a1] = y - bet * P
        else:
            V[a0:a1] = y
        vv = V[a0:a1].astype(np.float64)
        parts = [to_limbs((B.numpy()[i].reshape(n, n)[a0:a1].astype(np.float64) * vv).sum(axis=1)).sum(axis=0)
                 for i in range(m)]
        parts.append(to_limbs((vv * vv).sum(axis=1)).sum(axis=0))
        yy = y.astype(np.float64)
        parts.append(to_limbs((yy * yy).sum(axis=1)).sum(axis=0))
        self._add(dl[: 3 * (m + 2)], np.stack(parts))

    def update(self, v, B, m, dl, n, a0, a1, nl, scal):
        d = dl.numpy()
        h = [np.float32(from_limbs(*d[3 * i:3 * i + 3])) for i in range(m)]
        scal.numpy()[1] = np.sqrt(from_limbs(*d[3 * m + 3:3 * m + 6]))
        if a1 <= a0:
            return
        V = v.numpy().reshape(n, n)
        x = V[a0:a1].copy()
        for i in range(m):
            s = B.numpy()[i].reshape(n, n)[a0:a1]
            x = _fl32(x.astype(np.float64) - np.float64(h[i]) * s.astype(np.float64))
        V[a0:a1] = x
        xx = x.astype(np.float64)
        self._add(nl, to_limbs((xx * xx).sum(axis=1)).sum(axis=0))

    def normalize(self, src, nl, out, n, c, length, a0, a1, wl, scal):
        t = np.sqrt(from_limbs(*nl.numpy()))
        scal.numpy()[0] = t
        if a1 <= a0:
            return
        O = out.numpy().reshape(n, n)
        O[a0:a1] = src.numpy().reshape(n, n)[a0:a1] / np.float32(t)
        acc = np.zeros((length, 3), dtype=np.int64)
        for blk in range(a0, a1, 8):
            rows = O[blk:min(blk + 8, a1)].astype(np.float64)
            s = np.zeros(length)
            for r in range(rows.shape[0]):
                a = blk + r
                u = np.arange(n) - a + c
                ok = (u >= 0) & (u < length)
                s[u[ok]] += rows[r][ok]
            acc += to_limbs(s)
        self._add(wl[: 3 * length], acc)

    def lift(self, B, rows, W, out, off, ln, out_off=None):
        if ln == 0:
            return
        o = off if out_off is None else out_off
        out.numpy()[:, o:o + ln] = (W.numpy()[:rows].T.astype(np.float64)
                                    @ B.numpy()[:rows, off:off + ln].astype(np.float64)).astype(np.float32)
