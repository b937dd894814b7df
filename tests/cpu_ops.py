"""CPU stand-in for libfdmd used ONLY by the CPU test-suite to exercise the
host orchestration (sharding, all-reduces, pairing, table construction) on
machines without a GPU. It is a checker, never a product path: the package
has no CPU fallback and never imports this module."""

import numpy as np
import torch


def _logical(T):
    return T.view()


class CpuOps:
    def __init__(self):
        self.launches = 0

    def tall_gemm(self, A, B, C, stats=False, row_offset=0, alg_flops=None, upper=False, share_sms=False):
        K = B.shape[0]
        Av = _logical(A).to(torch.float64)
        if Av.shape[1] < K:  # row-major buffers may be multiplied over padded columns
            Av = A.buf[: A.n, :K].to(torch.float64)
        P = Av[:, :K] @ B.to(torch.float64)
        st = None
        if stats:
            N = P.shape[1]
            mag = P[:, 0::2] ** 2 + P[:, 1::2] ** 2
            st = torch.stack([mag.sum(0), mag.max(0).values, mag.argmax(0).to(torch.float64) + row_offset], dim=1)
            st = st[: N // 2]
        if C is not None:
            _logical(C).copy_(P.to(C.dtype))
        return st

    def tall_gram(self, A, B, K1=None, K2=None, symmetric=False, out=None, alg_flops=None, beta=0.0):
        Av = _logical(A).to(torch.float64)
        Bv = _logical(B).to(torch.float64)
        K1 = A.k if K1 is None else K1
        K2 = B.k if K2 is None else K2
        if A.layout == "col" and K1 > A.k:
            Av = A.buf[:K1, : A.n].t().to(torch.float64)
        G = Av[:, :K1].t() @ Bv[:, :K2]
        if out is not None:
            out.copy_(G if beta == 0.0 else beta * out + G)
            return out
        return G.contiguous()

    def tall_gram_bordered(self, A, K, out=None, beta=0.0, alg_flops=None):
        Av = _logical(A).to(torch.float64)
        G = Av[:, :K].t() @ Av[:, :K + 1]
        if out is not None:
            out.copy_(G if beta == 0.0 else beta * out + G)
            return out
        return G.contiguous()

    def tall_tdot(self, A, col, K, out=None, beta=0.0):
        Av = _logical(A).to(torch.float64)
        y = Av[:, :K].t() @ Av[:, col]
        if out is not None:
            out.copy_(beta * out + y)
            return out
        return y

    def decode(self, D, coef, out=None, ncols=None):
        r = D.k if ncols is None else ncols
        Dv = D.buf[:r, : D.n].to(torch.float64)
        res = (coef.to(torch.float64).t() @ Dv).to(D.dtype)
        if out is not None:
            out.copy_(res)
            return out
        return res

    def colmajor_dot(self, D, U, ncols=None):
        r = D.k if ncols is None else ncols
        return D.buf[:r, : D.n].to(torch.float64) @ U.to(torch.float64).t()

    def table_apply(self, R, src, alpha, beta, D, ncols):
        for j in range(ncols):
            u = src[j]
            v = alpha[j] * R.buf[2 * u, : R.n].to(torch.float64) + beta[j] * R.buf[2 * u + 1, : R.n].to(torch.float64)
            D.buf[j, : D.n] = v.to(D.dtype)

    def table_apply_inplace(self, R, src, alpha, beta, ncols):
        from paper_2502_05339_b200.device import Tall
        raw = R.buf[: R.k, : R.n].to(torch.float64).clone()
        for j in range(ncols):
            u = src[j]
            R.buf[j, : R.n] = (alpha[j] * raw[2 * u] + beta[j] * raw[2 * u + 1]).to(R.dtype)
        return Tall(R.buf, "col", R.n, ncols)

    def residual(self, S, D, F, ncols, T):
        Sv = _logical(S).to(torch.float64)
        rec = D.buf[:ncols, : D.n].to(torch.float64).t() @ F.to(torch.float64)
        e = Sv[:, 1:T + 1] - rec
        return torch.tensor([float((e * e).sum()), float((Sv[:, 1:T + 1] ** 2).sum())], dtype=torch.float64)

    def geev(self, K, vectors=True):
        w, V = np.linalg.eig(K.to(torch.float64).cpu().numpy())
        return (w, V) if vectors else (w, None)
