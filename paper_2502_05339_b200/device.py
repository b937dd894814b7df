"""Device plumbing: torch tensors for HBM buffers/streams/collectives, libfdmd
for every tall kernel.

Layout vocabulary (DESIGN.md §Data layout):
  * a ``Tall`` is an n x k matrix whose n (grid rows) is huge and k (snapshots,
    sketch width, modes) small. ``layout="row"``: buffer shape (n, ld), element
    (i, j) at buf[i, j] — snapshot matrices and sketches. ``layout="col"``:
    buffer shape (k, ld), element (i, j) at buf[j, i] — mode tables and bases,
    so a decode streams each mode column contiguously.
  * small factors (Omega, R^-1, W, Ub, ...) are plain fp64 torch tensors.

Row-sharding: when a ``Shard`` with world > 1 is attached, each rank holds a
contiguous row block and every reduction over n (tall_gram, colmajor_dot,
residual, pair statistics) is followed by one all-reduce of the small result.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import COL, F32, F64, ROW

_DT = {torch.float32: F32, torch.float64: F64}


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


@dataclass
class Tall:
    buf: torch.Tensor
    layout: str  # "row" | "col"
    n: int
    k: int

    @property
    def ld(self) -> int:
        return int(self.buf.shape[1])

    @property
    def dtype(self):
        return self.buf.dtype

    @property
    def code(self) -> int:
        return ROW if self.layout == "row" else COL

    def view(self) -> torch.Tensor:
        """Logical n x k view (may be a transposed view for col layout)."""
        if self.layout == "row":
            return self.buf[: self.n, : self.k]
        return self.buf[: self.k, : self.n].t()

    def nbytes(self) -> int:
        return self.buf.numel() * self.buf.element_size()


def alloc_tall(n: int, k: int, dtype, layout: str, device=None, zero: bool = False) -> Tall:
    device = device or torch.device("cuda", torch.cuda.current_device())
    elt = torch.empty((), dtype=dtype).element_size()
    q = 16 // elt
    if layout == "row":
        shape = (max(n, 1), round_up(max(k, 1), q))
    else:
        shape = (max(k, 1), round_up(max(n, 1), q))
    buf = (torch.zeros if zero else torch.empty)(shape, dtype=dtype, device=device)
    return Tall(buf, layout, n, k)


@dataclass
class Shard:
    """Row block [row0, row0 + n_local) of an n_global-row matrix."""

    row0: int
    n_local: int
    n_global: int
    group: object = None
    world: int = 1

    def _host_staged(self, t: torch.Tensor) -> bool:
        """gloo collectives on device tensors go through host memory (the CPU
        test harness and the 1-GPU multi-rank tests); NCCL reduces in HBM."""
        import torch.distributed as dist
        return t.is_cuda and dist.get_backend(self.group) == "gloo"

    def allreduce(self, t: torch.Tensor, op: str = "sum") -> torch.Tensor:
        """In-place all-reduce over the ranks' row blocks (sum or max)."""
        if self.world > 1:
            import torch.distributed as dist
            rop = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
            if self._host_staged(t):
                h = t.cpu()
                dist.all_reduce(h, op=rop, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=rop, group=self.group)
        return t

    def all_gather(self, t: torch.Tensor) -> list:
        """Every rank's copy of t, in rank order."""
        import torch.distributed as dist
        t = t.contiguous()
        if self._host_staged(t):
            h = t.cpu()
            out = [torch.empty_like(h) for _ in range(self.world)]
            dist.all_gather(out, h, group=self.group)
            return [o.to(t.device) for o in out]
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return out


SINGLE = None  # shard=None means the matrix is whole on this device


def allreduce(shard: Optional[Shard], t: torch.Tensor) -> torch.Tensor:
    return t if shard is None else shard.allreduce(t)


class _Workspace:
    def __init__(self):
        self.bufs = {}

    def get(self, nbytes: int, device) -> torch.Tensor:
        key = (str(device), torch.cuda.current_stream(device).cuda_stream)
        b = self.bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
            self.bufs[key] = b
        return b


class CudaOps:
    """Thin wrappers over libfdmd entry points. Counts kernel launches."""

    def __init__(self):
        self.ws = _Workspace()
        self.launches = 0
        self.profile = None   # list -> per-call (name, algorithmic flops, ev0, ev1)

    def _ev(self):
        if self.profile is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def _done(self, name, flops, e0, nbytes=0.0):
        """Record (name, algorithmic flops, ev0, ev1, algorithmic HBM bytes)."""
        if e0 is not None:
            self.profile.append((name, float(flops), e0, self._ev(), float(nbytes)))

    # -- C[n x N] = A * B (B small fp64, K x N) ---------------------------
    def tall_gemm(self, A: Tall, B: torch.Tensor, C: Optional[Tall], stats: bool = False,
                  row_offset: int = 0, alg_flops: Optional[float] = None,
                  upper: bool = False, share_sms: bool = False) -> Optional[torch.Tensor]:
        L = _lib.lib()
        K, N = int(B.shape[0]), int(B.shape[1])
        assert K <= A.k or K <= (A.ld if A.layout == "row" else K), (K, A.k)
        B = B.to(torch.float64).contiguous()
        st = None
        wsb = 0
        ws = None
        if stats:
            st = torch.empty((N // 2, 3), dtype=torch.float64, device=A.buf.device)
            wsb = int(L.fdmd_tall_gemm_workspace(A.n, N))
            ws = self.ws.get(wsb, A.buf.device)
        c_buf = C.buf if C is not None else None
        c_dt = _DT[C.dtype] if C is not None else F64
        c_lay = C.code if C is not None else COL
        c_ld = C.ld if C is not None else A.n
        e0 = self._ev()
        _lib.check(L.fdmd_tall_gemm(_ptr(A.buf), _DT[A.dtype], A.code, A.ld, _ptr(B), B.shape[1],
                                     _ptr(c_buf), c_dt, c_lay, c_ld, A.n, K, N,
                                     (1 if upper else 0) | (2 if share_sms else 0),
                                     _ptr(st), row_offset, _ptr(ws), wsb, _stream()), "tall_gemm")
        # algorithmic bytes: A read once, C written once (in place: read + write)
        nb = A.n * K * A.buf.element_size() + (A.n * N * C.buf.element_size() if C is not None else 0)
        self._done("tall_gemm", 2.0 * A.n * K * N if alg_flops is None else alg_flops, e0, nb)
        self.launches += 2 if stats else 1
        return st

    # -- C[K1 x K2] = A^T B over n ----------------------------------------
    def tall_gram(self, A: Tall, B: Tall, K1: Optional[int] = None, K2: Optional[int] = None,
                  symmetric: bool = False, out: Optional[torch.Tensor] = None,
                  alg_flops: Optional[float] = None, beta: float = 0.0) -> torch.Tensor:
        """out[K1 x K2] = beta * out + A^T B (fixed-order, deterministic)."""
        L = _lib.lib()
        K1 = A.k if K1 is None else K1
        K2 = B.k if K2 is None else K2
        if out is None:
            out = torch.empty((K1, K2), dtype=torch.float64, device=A.buf.device)
        wsb = int(L.fdmd_tall_gram_workspace(A.n, K1, K2))
        ws = self.ws.get(wsb, A.buf.device)
        e0 = self._ev()
        _lib.check(L.fdmd_tall_gram(_ptr(A.buf), _DT[A.dtype], A.code, A.ld, _ptr(B.buf), _DT[B.dtype],
                                     B.code, B.ld, _ptr(out), out.stride(0), float(beta), A.n, K1, K2,
                                     1 if symmetric else 0, _ptr(ws), wsb, _stream()), "tall_gram")
        if alg_flops is None:
            alg_flops = (1.0 if symmetric else 2.0) * A.n * K1 * K2
        nb = A.n * (K1 * A.buf.element_size() + (0 if symmetric else K2 * B.buf.element_size()))
        self._done("tall_gram", alg_flops, e0, nb)
        self.launches += 2
        return out

    # -- frames[f][i] = sum_k D[k][i] coef[k][f] ---------------------------
    def decode(self, D: Tall, coef: torch.Tensor, out: Optional[torch.Tensor] = None,
               ncols: Optional[int] = None) -> torch.Tensor:
        assert D.layout == "col"
        r = D.k if ncols is None else ncols
        coef = coef.to(D.dtype).contiguous()
        B = int(coef.shape[1])
        if out is None:
            out = torch.empty((B, D.n), dtype=D.dtype, device=D.buf.device)
        e0 = self._ev()
        _lib.check(_lib.lib().fdmd_decode(_ptr(D.buf), _DT[D.dtype], D.ld, _ptr(coef), coef.stride(0),
                                          _ptr(out), out.stride(0), D.n, r, B, _stream()), "decode")
        self._done("decode", 2.0 * D.n * r * B, e0)
        self.launches += (B + 31) // 32 if B > 16 else 1
        return out

    # -- tcgen05 batched reconstruction (FP16 2-way split) -----------------
    def tall_gram_bordered(self, A: Tall, K: int, out: Optional[torch.Tensor] = None, beta: float = 0.0,
                           alg_flops: Optional[float] = None) -> torch.Tensor:
        """out[K x (K+1)] = beta * out + [A[:, :K]^T A[:, :K] | A[:, :K]^T A[:, K]] in one
        pass over a row-major A (the snapshot Gram X^T X with the border X^T s_m)."""
        assert A.layout == "row" and K + 1 <= A.k
        L = _lib.lib()
        if out is None:
            out = torch.empty((K, K + 1), dtype=torch.float64, device=A.buf.device)
        wsb = int(L.fdmd_tall_gram_bordered_workspace(A.n, K))
        ws = self.ws.get(wsb, A.buf.device)
        e0 = self._ev()
        _lib.check(L.fdmd_tall_gram_bordered(_ptr(A.buf), _DT[A.dtype], A.ld, _ptr(out), out.stride(0), float(beta),
                                             A.n, K, _ptr(ws), wsb, _stream()), "tall_gram_bordered")
        if alg_flops is None:
            alg_flops = 1.0 * A.n * K * K + 2.0 * A.n * K
        self._done("tall_gram", alg_flops, e0, A.n * (K + 1) * A.buf.element_size())
        self.launches += 2
        return out

    def tall_tdot(self, A: Tall, col: int, K: int, out: Optional[torch.Tensor] = None,
                  beta: float = 0.0) -> torch.Tensor:
        """y (K, f64) = A[:, :K]^T A[:, col] over the rows of a row-major A (the
        border X^T s_m of the snapshot Gram); out = beta*out + y when given."""
        assert A.layout == "row" and 0 <= col < A.k and K <= A.k
        L = _lib.lib()
        y = torch.zeros((K,), dtype=torch.float64, device=A.buf.device) if out is None else out
        wsb = int(L.fdmd_tall_tdot_workspace(A.n, K))
        ws = self.ws.get(wsb, A.buf.device)
        e0 = self._ev()
        vp = A.buf.data_ptr() + col * A.buf.element_size()
        _lib.check(L.fdmd_tall_tdot(_ptr(A.buf), _DT[A.dtype], A.ld, ctypes.c_void_p(vp), A.ld, A.n, K, _ptr(y),
                                    float(beta if out is not None else 0.0), _ptr(ws), wsb, _stream()), "tall_tdot")
        self._done("tall_tdot", 2.0 * A.n * K, e0, A.n * A.ld * A.buf.element_size())
        self.launches += 2
        return y

    def tall_gemm_planes(self, A: Tall, B: torch.Tensor, bound: float = 2.0, alg_flops: Optional[float] = None,
                         share_sms: bool = False) -> dict:
        """A @ B on FP64 DMMA written straight into the fp16 hi/lo planes
        tc_decode streams (row-major n x round_up(N, 8)); `bound` = a known
        max |A @ B| (orthonormal columns: <= 1) fixes the plane scale."""
        import math
        assert A.layout == "row"
        K, N = int(B.shape[0]), int(B.shape[1])
        B = B.to(torch.float64).contiguous()
        ldu = round_up(N, 8)
        su = math.ldexp(1.0, 14 - math.frexp(float(bound))[1])
        uh = torch.empty((A.n, ldu), dtype=torch.float16, device=A.buf.device)
        ul = torch.empty_like(uh)
        e0 = self._ev()
        _lib.check(_lib.lib().fdmd_tall_gemm_planes(_ptr(A.buf), _DT[A.dtype], A.ld, _ptr(B), N, _ptr(uh), _ptr(ul),
                                                    ldu, float(su), A.n, K, N, 2 if share_sms else 0, _stream()),
                   "tall_gemm_planes")
        self._done("tall_gemm", 2.0 * A.n * K * N if alg_flops is None else alg_flops, e0,
                   A.n * K * A.buf.element_size() + 4 * A.n * ldu)
        return {"uh": uh, "ul": ul, "ldu": ldu, "su": su, "n": A.n, "r": N}

    def tc_basis(self, D: Tall, ncols: Optional[int] = None, bound: Optional[float] = None):
        """Split a column-major fp32 basis into the row-major fp16 hi/lo
        planes the tcgen05 kernel streams (built once per basis). `bound`: a
        known max |D| (orthonormal columns: <= 1) skips the scan and its sync."""
        import math
        assert D.layout == "col" and D.dtype == torch.float32
        r = D.k if ncols is None else ncols
        n = D.n
        ldu = round_up(r, 8)
        if bound is not None:
            mx = float(bound)
        elif n:   # one read pass, no |U| temporary (a 40 GB abs() copy at config 4)
            lo, hi = torch.aminmax(D.buf[:r, :n])
            mx = max(-float(lo.item()), float(hi.item()))
        else:
            mx = 0.0
        e = math.frexp(mx)[1] if mx > 0 else 0
        su = math.ldexp(1.0, 14 - e)
        uh = torch.empty((n, ldu), dtype=torch.float16, device=D.buf.device)
        ul = torch.empty_like(uh)
        _lib.check(_lib.lib().fdmd_split_basis(_ptr(D.buf), D.ld, n, r, ctypes.c_float(su), _ptr(uh), _ptr(ul),
                                               ldu, _stream()), "split_basis")
        self.launches += 1
        return {"uh": uh, "ul": ul, "ldu": ldu, "su": su, "n": n, "r": r}

    def tc_rows(self, A: Tall, ncols: Optional[int] = None, bound: Optional[float] = None):
        """fp16 hi/lo planes of a row-major fp64 tall matrix (the sketch basis
        Q) for tc_decode: products Q @ M on tcgen05, FP32-accurate. `bound`:
        a known max |A| (an orthonormal basis: ~1) skips the scan and its host
        sync, so the launch overlaps host-side small work."""
        import math
        assert A.layout == "row" and A.dtype in (torch.float64, torch.float32)
        K = A.k if ncols is None else ncols
        n = A.n
        ldu = round_up(K, 8)
        if bound is not None:
            mx = float(bound)
        else:
            lo, hi = torch.aminmax(A.buf[:n, :K])
            mx = max(-float(lo.item()), float(hi.item()))
        e = math.frexp(mx)[1] if mx > 0 else 0
        su = math.ldexp(1.0, 14 - e)
        uh = torch.empty((n, ldu), dtype=torch.float16, device=A.buf.device)
        ul = torch.empty_like(uh)
        _lib.check(_lib.lib().fdmd_split_rows(_ptr(A.buf), _DT[A.dtype], A.ld, n, K, float(su), _ptr(uh), _ptr(ul),
                                              ldu, _stream()), "split_rows")
        self.launches += 1
        return {"uh": uh, "ul": ul, "ldu": ldu, "su": su, "n": n, "r": K}

    def pair_stats(self, raw: Tall, units: int, row_offset: int = 0) -> torch.Tensor:
        """(units, 3) [sum |phi|^2, max |phi|^2, argmax row] of a col-major fp32 table."""
        assert raw.layout == "col" and raw.dtype == torch.float32
        L = _lib.lib()
        out = torch.empty((units, 3), dtype=torch.float64, device=raw.buf.device)
        wsb = int(L.fdmd_pair_stats_workspace(raw.n, units))
        ws = self.ws.get(wsb, raw.buf.device)
        _lib.check(L.fdmd_pair_stats(_ptr(raw.buf), raw.ld, raw.n, units, int(row_offset), _ptr(out), _ptr(ws), wsb,
                                     _stream()), "pair_stats")
        self.launches += 2
        return out

    def tc_decode(self, tcb: dict, coef: torch.Tensor, out: Optional[torch.Tensor] = None,
                  share_sms: bool = False) -> torch.Tensor:
        """frames (B x n fp32) = basis @ coef (r x B) on tcgen05."""
        r, n = tcb["r"], tcb["n"]
        coef = coef.to(torch.float32).contiguous()
        B = int(coef.shape[1])
        ldk = round_up(r, 8)
        dev = coef.device
        ch = torch.empty((B, ldk), dtype=torch.float16, device=dev)
        cl = torch.empty_like(ch)
        fs = torch.empty((B,), dtype=torch.float32, device=dev)
        if out is None:
            out = torch.empty((B, n), dtype=torch.float32, device=dev)
        e0 = self._ev()
        L = _lib.lib()
        _lib.check(L.fdmd_split_coef(_ptr(coef), coef.stride(0), r, B, ctypes.c_float(1.0 / tcb["su"]), _ptr(ch),
                                     _ptr(cl), ldk, _ptr(fs), _stream()), "split_coef")
        _lib.check(L.fdmd_tc_decode_ex(_ptr(tcb["uh"]), _ptr(tcb["ul"]), tcb["ldu"], n, r, _ptr(ch), _ptr(cl), ldk,
                                       B, _ptr(fs), _ptr(out), out.stride(0), 2 if share_sms else 0, _stream()),
                   "tc_decode")
        self._done("tc_decode", 2.0 * n * r * B, e0)
        self.launches += 2
        return out

    def tc_decode_pairstats(self, tcb: dict, coef: torch.Tensor, out: torch.Tensor, units: int,
                            row_offset: int = 0) -> Optional[torch.Tensor]:
        """tc_decode of a modes product (columns 2u, 2u+1 = Re, Im of mode u) whose
        frame epilogue also takes max_i |phi_u[i]|^2 and the first row attaining it
        and the sum of |phi_u|^2 (the statistics pair_stats reads back from the
        table). Returns st (units x 3 f64) or None when the batch is too narrow for
        the CTA-pair kernel (the frames are still written)."""
        r, n = tcb["r"], tcb["n"]
        coef = coef.to(torch.float32).contiguous()
        B = int(coef.shape[1])
        assert B == 2 * units
        ldk = round_up(r, 8)
        dev = coef.device
        ch = torch.empty((B, ldk), dtype=torch.float16, device=dev)
        cl = torch.empty_like(ch)
        fs = torch.empty((B,), dtype=torch.float32, device=dev)
        st = torch.zeros((units, 3), dtype=torch.float64, device=dev)
        fused = ctypes.c_int(0)
        e0 = self._ev()
        L = _lib.lib()
        _lib.check(L.fdmd_split_coef(_ptr(coef), coef.stride(0), r, B, ctypes.c_float(1.0 / tcb["su"]), _ptr(ch),
                                     _ptr(cl), ldk, _ptr(fs), _stream()), "split_coef")
        _lib.check(L.fdmd_tc_decode_pairstats(_ptr(tcb["uh"]), _ptr(tcb["ul"]), tcb["ldu"], n, r, _ptr(ch), _ptr(cl),
                                              ldk, B, _ptr(fs), _ptr(out), out.stride(0), int(row_offset), _ptr(st),
                                              ctypes.byref(fused), _stream()), "tc_decode_pairstats")
        self._done("tc_decode", 2.0 * n * r * B, e0)
        self.launches += 3 if fused.value else 2
        return st if fused.value else None

    def tc_decode_planes(self, tcb: dict, coef: torch.Tensor, bound: float = 2.0, share_sms: bool = False) -> dict:
        """basis @ coef (r x k, k <= 256) on tcgen05, written straight into the
        fp16 hi/lo planes of a row-major n x round_up(k, 8) matrix (the lift
        U = Q Ub into the config-4 basis planes: no fp32 U, no separate split).
        `bound`: a known max |result| (orthonormal columns: <= 1) fixes the
        plane scale su = 2^(14 - e) without a scan."""
        import math
        r, n = tcb["r"], tcb["n"]
        coef = coef.to(torch.float32).contiguous()
        k = int(coef.shape[1])
        ldk = round_up(r, 8)
        ldp = round_up(k, 8)
        dev = coef.device
        ch = torch.empty((k, ldk), dtype=torch.float16, device=dev)
        cl = torch.empty_like(ch)
        fs = torch.empty((k,), dtype=torch.float32, device=dev)
        e = math.frexp(float(bound))[1]
        su = math.ldexp(1.0, 14 - e)
        uh = torch.empty((n, ldp), dtype=torch.float16, device=dev)
        ul = torch.empty_like(uh)
        e0 = self._ev()
        L = _lib.lib()
        _lib.check(L.fdmd_split_coef(_ptr(coef), coef.stride(0), r, k, ctypes.c_float(1.0 / tcb["su"]), _ptr(ch),
                                     _ptr(cl), ldk, _ptr(fs), _stream()), "split_coef")
        _lib.check(L.fdmd_tc_decode_planes(_ptr(tcb["uh"]), _ptr(tcb["ul"]), tcb["ldu"], n, r, _ptr(ch), _ptr(cl),
                                           ldk, k, _ptr(fs), _ptr(uh), _ptr(ul), ldp, ctypes.c_float(su),
                                           2 if share_sms else 0, _stream()), "tc_decode_planes")
        self._done("tc_decode", 2.0 * n * r * k, e0)
        self.launches += 2
        return {"uh": uh, "ul": ul, "ldu": ldp, "su": su, "n": n, "r": k}

    # -- y[k][v] = sum_i D[k][i] U[v][i] -----------------------------------
    def colmajor_dot(self, D: Tall, U: torch.Tensor, ncols: Optional[int] = None) -> torch.Tensor:
        """U: (nv, n) tensor (nv <= 8), row v contiguous."""
        assert D.layout == "col"
        L = _lib.lib()
        r = D.k if ncols is None else ncols
        if U.dtype not in (torch.float32, torch.float64):
            U = U.to(torch.float64)
        U = U.contiguous()
        nv = int(U.shape[0])
        y = torch.empty((r, nv), dtype=torch.float64, device=D.buf.device)
        wsb = int(L.fdmd_colmajor_dot_workspace(D.n, r, nv))
        ws = self.ws.get(wsb, D.buf.device)
        _lib.check(L.fdmd_colmajor_dot(_ptr(D.buf), _DT[D.dtype], D.ld, _ptr(U), _DT[U.dtype], U.stride(0),
                                       D.n, r, nv, _ptr(y), _ptr(ws), wsb, _stream()), "colmajor_dot")
        self.launches += 2
        return y

    # -- 2-D MAC grids: serving / guided upscaling --------------------------
    def mac_decode(self, D: Tall, coef: torch.Tensor, nx: int, ny: int, field: str,
                   ncols: Optional[int] = None) -> torch.Tensor:
        """Cell-centred planes (f64, (2|1) x ny x nx) of the decoded state."""
        assert D.layout == "col"
        r = int(coef.numel()) if ncols is None else ncols
        coef = coef.reshape(-1).to(device=D.buf.device, dtype=torch.float64).contiguous()
        code = {"velocity": 0, "speed": 1}[field]
        out = torch.empty((2 if code == 0 else 1, ny, nx), dtype=torch.float64, device=D.buf.device)
        _lib.check(_lib.lib().fdmd_mac_decode(_ptr(D.buf), _DT[D.dtype], D.ld, r, _ptr(coef), nx, ny, code,
                                              _ptr(out), _stream()), "mac_decode")
        self.launches += 1
        return out

    def mac_advect(self, vel: torch.Tensor, nx: int, ny: int, h: float, dt: float,
                   q: torch.Tensor) -> torch.Tensor:
        """One semi-Lagrangian step of the cell-centred scalar q (ny x nx f64)."""
        vel = vel.reshape(-1).contiguous()
        if vel.dtype not in (torch.float32, torch.float64):
            vel = vel.to(torch.float64)
        q = q.to(torch.float64).contiguous()
        out = torch.empty_like(q)
        _lib.check(_lib.lib().fdmd_mac_advect(_ptr(vel), _DT[vel.dtype], nx, ny, float(h), float(dt), _ptr(q),
                                              _ptr(out), _stream()), "mac_advect")
        self.launches += 1
        return out

    def mac_inject(self, low: torch.Tensor, nx: int, ny: int, factor: int) -> torch.Tensor:
        """(nv, n_state_high) fine states from (nv, n_state_low) coarse states."""
        low = low.to(torch.float64)
        if low.dim() == 1:
            low = low[None, :]
        low = low.contiguous()
        nh = (nx + 1) * ny + nx * (ny + 1)
        fine = torch.empty((low.shape[0], nh), dtype=torch.float64, device=low.device)
        _lib.check(_lib.lib().fdmd_mac_inject(_ptr(low), nx, ny, factor, int(low.shape[0]), low.stride(0),
                                              fine.stride(0), _ptr(fine), _stream()), "mac_inject")
        self.launches += 1
        return fine

    def mac_project(self, H: torch.Tensor, L: torch.Tensor, nx: int, ny: int, factor: int,
                    gram_diag: float) -> torch.Tensor:
        H = H.reshape(-1).to(torch.float64).contiguous()
        L = L.reshape(-1).to(device=H.device, dtype=torch.float64).contiguous()
        x = torch.empty_like(H)
        _lib.check(_lib.lib().fdmd_mac_project(_ptr(H), _ptr(L), nx, ny, factor, float(gram_diag), _ptr(x),
                                               _stream()), "mac_project")
        self.launches += 1
        return x

    def table_apply(self, R: Tall, src, alpha, beta, D: Tall, ncols: int):
        dev = R.buf.device
        src_t = torch.as_tensor(np.asarray(src, dtype=np.int32), device=dev)
        a_t = torch.as_tensor(np.asarray(alpha, dtype=np.float64), device=dev)
        b_t = torch.as_tensor(np.asarray(beta, dtype=np.float64), device=dev)
        _lib.check(_lib.lib().fdmd_table_apply(_ptr(R.buf), _DT[R.dtype], R.ld, _ptr(src_t), _ptr(a_t),
                                               _ptr(b_t), _ptr(D.buf), _DT[D.dtype], D.ld, D.n, ncols,
                                               _stream()), "table_apply")
        self.launches += 1

    def table_apply_inplace(self, R: Tall, src, alpha, beta, ncols: int) -> Tall:
        """R's first ncols columns become the table (R column-major, 2U >= ncols)."""
        dev = R.buf.device
        src_t = torch.as_tensor(np.asarray(src, dtype=np.int32), device=dev)
        a_t = torch.as_tensor(np.asarray(alpha, dtype=np.float64), device=dev)
        b_t = torch.as_tensor(np.asarray(beta, dtype=np.float64), device=dev)
        _lib.check(_lib.lib().fdmd_table_apply_inplace(_ptr(R.buf), _DT[R.dtype], R.ld, R.k, _ptr(src_t),
                                                       _ptr(a_t), _ptr(b_t), ncols, R.n, _stream()),
                   "table_apply_inplace")
        self.launches += 1
        return Tall(R.buf, "col", R.n, ncols)

    def residual(self, S: Tall, D: Tall, F: torch.Tensor, ncols: int, T: int) -> torch.Tensor:
        L = _lib.lib()
        F = F.to(torch.float64).contiguous()
        out = torch.empty((2,), dtype=torch.float64, device=S.buf.device)
        wsb = int(L.fdmd_residual_workspace(S.n))
        ws = self.ws.get(wsb, S.buf.device)
        _lib.check(L.fdmd_residual(_ptr(S.buf), _DT[S.dtype], S.ld, _ptr(D.buf), _DT[D.dtype], D.ld,
                                   _ptr(F), ncols, T, S.n, _ptr(out), _ptr(ws), wsb, _stream()), "residual")
        self.launches += 2
        return out

    def svd_small(self, B: torch.Tensor):
        """Thin SVD of the small device matrix B (l x T, l <= T): (Ub, s, Vh, info)
        with info a device int32 (cuSOLVER gesvdp's status; 0 = converged).
        Stream-ordered on the current stream, no host synchronisation."""
        l, T = int(B.shape[0]), int(B.shape[1])
        assert l <= T and B.is_cuda
        A = B.to(torch.float64).clone(memory_format=torch.contiguous_format)
        dev = B.device
        ubt = torch.empty((l, l), dtype=torch.float64, device=dev)
        sv = torch.empty((l,), dtype=torch.float64, device=dev)
        vh = torch.empty((l, T), dtype=torch.float64, device=dev)
        info = torch.zeros((), dtype=torch.int32, device=dev)
        _lib.check(_lib.lib().fdmd_svd_small(_ptr(A), A.stride(0), l, T, _ptr(ubt), _ptr(sv), _ptr(vh), _ptr(info),
                                             _stream()), "svd_small")
        return ubt.t(), sv, vh, info

    def geev(self, K: torch.Tensor, vectors: bool = True):
        """Real nonsymmetric eig on device (cuSOLVER Xgeev). Returns host
        (w complex[n], V complex[n, n]) with LAPACK pair unpacking; V is None
        when vectors=False (eigenvalues only)."""
        n = int(K.shape[0])
        A = K.to(torch.float64).t().contiguous().clone()  # column-major
        w = np.empty(2 * n, dtype=np.float64)
        vr = np.empty(n * n, dtype=np.float64) if vectors else None
        _lib.check(_lib.lib().fdmd_geev(n, _ptr(A), w.ctypes.data_as(ctypes.c_void_p),
                                        vr.ctypes.data_as(ctypes.c_void_p) if vectors else None,
                                        _stream()), "geev")
        lam = w[0::2] + 1j * w[1::2]
        if not vectors:
            return lam, None
        VR = vr.reshape(n, n).T  # column-major -> (row, col)
        V = np.empty((n, n), dtype=np.complex128)
        j = 0
        while j < n:
            if lam[j].imag != 0.0 and j + 1 < n:
                V[:, j] = VR[:, j] + 1j * VR[:, j + 1]
                V[:, j + 1] = VR[:, j] - 1j * VR[:, j + 1]
                j += 2
            else:
                V[:, j] = VR[:, j]
                j += 1
        return lam, V

    def synth3d(self, tables, m: int, noise: float, key: int, row0: int, rows: int, out: Tall):
        sx, sy, sz, A = tables
        K, C, N = int(sx.shape[0]), int(sx.shape[1]), int(sx.shape[2])
        _lib.check(_lib.lib().fdmd_synth3d(_ptr(sx), _ptr(sy), _ptr(sz), _ptr(A), K, C, N, m, noise,
                                           ctypes.c_uint64(key), row0, rows, _ptr(out.buf), _DT[out.dtype],
                                           out.ld, _stream()), "synth3d")
        self.launches += 1


ops = CudaOps()


def set_ops(o):
    """Swap the kernel provider (tests use this to run the host orchestration
    with a CPU checker). Returns the previous provider."""
    global ops
    prev, ops = ops, o
    return prev


def get_ops():
    return ops


def default_device():
    if not torch.cuda.is_available():
        raise _lib.DeviceError("no CUDA device: the DMD hot path runs only on the GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())
