"""Model files and dataset directories for device-resident models.

SURVEY.md §8(f) row 1 — the callers' on-disk formats of the reference
(model_io.py:46-336, docs/formats.md:35-92), byte-compatible in both
directions:

* model file: ``KDMD`` | u32 version | u64 n | u64 r | f64 dt | u32 len +
  grid key=value block | r f64 sigma | r c128 lambda | n*r c128 phi
  (column-major) | u32 len + provenance block | u32 CRC32 of everything
  before it (model_io.py:154-181);
* dataset directory: ``manifest`` (key = value text) + ``snapshots.bin``
  (f64, column-major n x frames) [+ ``density.bin``] (model_io.py:258-336).

B200 design: phi (161 GB at config 3) and the snapshots never pass through
host memory whole. ``save_model`` forms phi a few modes at a time on the
device from the decode table (phi = D E) and streams c128 blocks through a
pinned buffer into the file with a running CRC32; ``load_model`` streams the
file back, validating sizes first and the CRC before returning, and writes
the table columns straight into HBM. Datasets move in blocks of 8 columns,
transposed on the device between the file's column-major layout and the
row-major HBM layout the kernels read.
"""

from __future__ import annotations

import dataclasses
import os
import zlib
from typing import Optional

import numpy as np
import torch

from . import device as dv
from .device import alloc_tall
from .grid import GridSpec  # noqa: F401  (re-export)
from .errors import BadMagicError, BadVersionError, ChecksumError, SizeMismatchError

MAGIC = b"KDMD"
VERSION = 1
_U32 = np.dtype("<u4")
_U64 = np.dtype("<u8")
_F64 = np.dtype("<f8")
_C128 = np.dtype("<c16")

MANIFEST_NAME = "manifest"
SNAPSHOTS_NAME = "snapshots.bin"
DENSITY_NAME = "density.bin"

BLOCK_MODES = 4      # phi columns formed / transferred per step
BLOCK_COLS = 8       # snapshot columns per dataset transfer


# ---------------------------------------------------------------------------
# key = value text codec (model_io.py:46-104)
# ---------------------------------------------------------------------------
def format_value(value) -> str:
    """Canonical text of a scalar or flat list (model_io.py:76-90)."""
    if isinstance(value, str):
        return value
    if isinstance(value, (bool, np.bool_)):
        return "true" if value else "false"
    if value is None:
        return "none"
    if isinstance(value, (int, np.integer)):
        return str(int(value))
    if isinstance(value, (float, np.floating)):
        return repr(float(value))
    if isinstance(value, (list, tuple, np.ndarray)):
        return ",".join(format_value(v) for v in np.asarray(value).ravel().tolist())
    return str(value)


def kv_dumps(pairs) -> str:
    out = []
    for key, value in pairs.items():
        key, value = str(key), format_value(value)
        if "=" in key or "\n" in key:
            raise ValueError(f"illegal key {key!r}")
        if "\n" in value:
            raise ValueError(f"value for {key!r} contains a newline")
        out.append(f"{key} = {value}")
    return "\n".join(out) + "\n"


def kv_loads(text: str) -> dict:
    out = {}
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise ValueError(f"line {lineno}: expected 'key = value', got {raw!r}")
        key, _, value = line.partition("=")
        out[key.strip()] = value.strip()
    return out


def parse_bool(text: str) -> bool:
    if text == "true":
        return True
    if text == "false":
        return False
    raise ValueError(f"expected true/false, got {text!r}")


def parse_floats(text: str) -> np.ndarray:
    if text.strip() == "":
        return np.zeros(0)
    return np.array([float(v) for v in text.split(",")])


# ---------------------------------------------------------------------------
# grid metadata block (model_io.py:107-140)
# ---------------------------------------------------------------------------
# GridSpec lives in grid.py (reference grid.py:27-97); re-exported here.


def grid_to_kv(grid) -> dict:
    if grid is None:
        return {"kind": "none"}
    if all(hasattr(grid, a) for a in ("nx", "ny", "h", "boundary")):   # ours or the reference's GridSpec
        out = {"kind": "grid", "nx": grid.nx, "ny": grid.ny, "h": grid.h, "boundary": grid.boundary}
        solids = np.flatnonzero(np.asarray(grid.solids()).ravel()) if hasattr(grid, "solids") else []
        if len(solids):
            out["solid_cells"] = list(solids)
        return out
    raise ValueError(f"cannot serialize grid metadata of type {type(grid).__name__}")


def grid_from_kv(kv: dict):
    kind = kv.get("kind", "none")
    if kind == "none":
        return None
    if kind != "grid":
        raise ValueError(f"unknown grid block kind {kind!r}")
    nx, ny = int(kv["nx"]), int(kv["ny"])
    mask = None
    if "solid_cells" in kv:
        mask = np.zeros(nx * ny, dtype=bool)
        mask[[int(v) for v in kv["solid_cells"].split(",")]] = True
        mask = mask.reshape(ny, nx)
    return GridSpec(nx, ny, float(kv["h"]), kv["boundary"], mask)


# ---------------------------------------------------------------------------
# model files (model_io.py:154-251)
# ---------------------------------------------------------------------------
def _u32(v) -> bytes:
    return np.asarray([v], dtype=_U32).tobytes()


def _u64(v) -> bytes:
    return np.asarray([v], dtype=_U64).tobytes()


class _CrcFile:
    def __init__(self, fh):
        self.fh, self.crc = fh, 0

    def write(self, b):
        self.crc = zlib.crc32(b, self.crc)
        self.fh.write(b)


def _pinned(shape, dtype):
    return torch.empty(shape, dtype=dtype, pin_memory=torch.cuda.is_available())


def _stream_out(fh, crc: int, blocks, rows_max: int, n: int, dtype) -> int:
    """Write device blocks (rows x n) to `fh` in order with a running CRC32.
    Double-buffered pinned staging: a writer thread (zlib.crc32 and the file
    write release the GIL) drains block i while the caller forms block i+1
    on the device and copies it down."""
    from concurrent.futures import ThreadPoolExecutor
    bufs = [_pinned((rows_max, n), dtype) for _ in range(2)]
    state = {"crc": crc}

    def sink(mv):
        state["crc"] = zlib.crc32(mv, state["crc"])
        fh.write(mv)

    pend = [None, None]
    with ThreadPoolExecutor(1) as ex:
        for i, blk in enumerate(blocks):
            b = i & 1
            if pend[b] is not None:
                pend[b].result()
            hv = bufs[b][: blk.shape[0]]
            hv.copy_(blk, non_blocking=True)
            if blk.is_cuda:
                torch.cuda.current_stream(blk.device).synchronize()
            pend[b] = ex.submit(sink, memoryview(hv.numpy()).cast("B"))
        for f in pend:
            if f is not None:
                f.result()
    return state["crc"]


def _stream_in(fh, crc: int, rows: list, n: int, dtype, consume):
    """Read consecutive blocks (rows[i] x n) from `fh` with a running CRC32:
    a reader thread fills the other pinned buffer while `consume(i, host)`
    uploads the current one. Stops early when consume returns False.
    Returns (crc, completed)."""
    from concurrent.futures import ThreadPoolExecutor
    bufs = [_pinned((max(rows), n), dtype) for _ in range(2)]
    state = {"crc": crc}

    def fill(b, k):
        hv = bufs[b][:k]
        mv = memoryview(hv.numpy()).cast("B")
        fh.readinto(mv)
        state["crc"] = zlib.crc32(mv, state["crc"])
        return hv

    with ThreadPoolExecutor(1) as ex:
        fut = ex.submit(fill, 0, rows[0])
        for i, k in enumerate(rows):
            hv = fut.result()
            if i + 1 < len(rows):
                fut = ex.submit(fill, (i + 1) & 1, rows[i + 1])
            if consume(i, hv) is False:
                if i + 1 < len(rows):
                    fut.result()
                return state["crc"], False
    return state["crc"], True


def _phi_block(model, a0: int, a1: int) -> torch.Tensor:
    """phi[:, a0:a1] transposed (b x n complex128, device), from the table."""
    modes = model.modes
    D, E = modes.basis()
    Eb = E[:, a0:a1]
    C = np.concatenate([Eb.real, Eb.imag], axis=1)                     # nraw x 2b
    dev = D.buf.device
    fr = dv.get_ops().decode(D, torch.as_tensor(C, device=dev), ncols=E.shape[0]).to(torch.float64)
    b = a1 - a0
    return torch.complex(fr[:b], fr[b:])


def _gathered_phi_blocks(model, shard):
    """Row-sharded model: each block of phi columns is formed on every rank
    from its table rows and gathered in rank (= row) order; yields the full
    (b x n) blocks on every rank (rank 0 writes them)."""
    n_max = max(shard.all_gather(torch.tensor([model.modes.n_local], device=model.modes.table.buf.device)))
    n_max = int(n_max.item())
    for a0 in range(0, model.r, BLOCK_MODES):
        blk = _phi_block(model, a0, min(model.r, a0 + BLOCK_MODES))                    # b x n_loc
        pad = torch.zeros((blk.shape[0], n_max), dtype=blk.dtype, device=blk.device)
        pad[:, : blk.shape[1]] = blk
        parts = shard.all_gather(torch.view_as_real(pad))
        sizes = shard.all_gather(torch.tensor([blk.shape[1]], device=blk.device))
        yield torch.cat([torch.view_as_complex(p)[:, : int(k.item())] for p, k in zip(parts, sizes)], dim=1)


def save_model(path, model):
    """Write ``model`` in the reference's model-file format
    (model_io.py:154-181), phi streamed from the device table. A row-sharded
    model is written by rank 0 with every rank's rows gathered block by block
    (a collective: every rank of the shard group calls it)."""
    m = model.modes
    shard = m.shard if (m.shard is not None and m.shard.world > 1) else None
    if shard is not None:
        import torch.distributed as dist
        rank = dist.get_rank(shard.group)
        if rank != 0:
            for _ in _gathered_phi_blocks(model, shard):
                pass
            dist.barrier(group=shard.group)
            return
    n, r = model.n, model.r
    grid_block = kv_dumps(grid_to_kv(model.grid_meta)).encode("utf-8")
    prov_block = kv_dumps({str(k): format_value(v) for k, v in sorted(model.provenance.items())}).encode("utf-8")
    tmp = f"{path}.tmp"
    with open(tmp, "wb") as fh:
        w = _CrcFile(fh)
        w.write(MAGIC + _u32(VERSION) + _u64(n) + _u64(r) + np.asarray([model.dt], dtype=_F64).tobytes())
        w.write(_u32(len(grid_block)) + grid_block)
        w.write(np.ascontiguousarray(model.sigma, dtype=_F64).tobytes())
        w.write(np.ascontiguousarray(model.lam, dtype=_C128).tobytes())
        if shard is None:
            blocks = (_phi_block(model, a0, min(r, a0 + BLOCK_MODES)) for a0 in range(0, r, BLOCK_MODES))
        else:
            blocks = _gathered_phi_blocks(model, shard)
        w.crc = _stream_out(fh, w.crc, blocks, BLOCK_MODES, n, torch.complex128)   # (b, n) c128 = phi columns
        w.write(_u32(len(prov_block)) + prov_block)
        fh.write(_u32(w.crc))
    os.replace(tmp, path)
    if shard is not None:
        import torch.distributed as dist
        dist.barrier(group=shard.group)


def _read_exact(fh, count, what, offset, total):
    if offset + count > total:
        raise SizeMismatchError(f"file truncated while reading {what} "
                                f"(need {count} bytes at offset {offset}, have {total - offset})")
    b = fh.read(count)
    return b


def load_model(path, device=None, table_dtype=torch.float64):
    """Read and validate a model file (model_io.py:206-251) into a
    device-resident ReducedModel: BadMagicError, BadVersionError,
    SizeMismatchError (truncated / trailing bytes) and ChecksumError as the
    reference. phi streams from disk into the HBM decode table."""
    from .dmd import ReducedModel
    from .modes import DeviceModes, conjugate_pairs
    dev = device or dv.default_device()
    total = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(4)
        if len(head) < 4 or head != MAGIC:
            raise BadMagicError(f"{path}: not a model file (bad magic)")
        crc = zlib.crc32(head)
        pos = 4

        def take(count, what):
            nonlocal pos, crc
            b = _read_exact(fh, count, what, pos, total)
            pos += count
            crc = zlib.crc32(b, crc)
            return b

        version = int(np.frombuffer(take(4, "version"), dtype=_U32)[0])
        if version != VERSION:
            raise BadVersionError(f"{path}: unsupported version {version}")
        n = int(np.frombuffer(take(8, "n"), dtype=_U64)[0])
        r = int(np.frombuffer(take(8, "r"), dtype=_U64)[0])
        dt = float(np.frombuffer(take(8, "dt"), dtype=_F64)[0])
        glen = int(np.frombuffer(take(4, "grid block length"), dtype=_U32)[0])
        grid_raw = take(glen, "grid block")
        sigma = np.frombuffer(take(8 * r, "sigma"), dtype=_F64).copy()
        lam = np.frombuffer(take(16 * r, "lambda"), dtype=_C128).copy()
        phi_off = pos
        # structure first (the reference reads the blob, then checks sizes): peek
        # at the provenance length behind phi without reading phi
        if phi_off + 16 * n * r > total:
            raise SizeMismatchError(f"file truncated while reading phi (need {16 * n * r} bytes at offset "
                                    f"{phi_off}, have {total - phi_off})")
        fh.seek(phi_off + 16 * n * r)
        plen_raw = fh.read(4)
        if len(plen_raw) < 4:
            raise SizeMismatchError(f"file truncated while reading provenance length (need 4 bytes at offset "
                                    f"{phi_off + 16 * n * r}, have {len(plen_raw)})")
        plen = int(np.frombuffer(plen_raw, dtype=_U32)[0])
        payload_len = phi_off + 16 * n * r + 4 + plen
        if payload_len > total:
            raise SizeMismatchError(f"file truncated while reading provenance block (need {plen} bytes at offset "
                                    f"{payload_len - plen}, have {total - payload_len + plen})")
        if payload_len + 4 > total:
            raise SizeMismatchError(f"file truncated while reading crc32 (need 4 bytes at offset {payload_len}, "
                                    f"have {total - payload_len})")
        if payload_len + 4 != total:
            raise SizeMismatchError(f"{path}: {total - payload_len - 4} trailing bytes after checksum")
        # stream phi (column-major: mode after mode) into the device table
        fh.seek(phi_off)
        crc_head = crc
        partner = conjugate_pairs(lam)
        adjacent = all(partner[a] in (a, a + 1, a - 1) for a in range(r))
        builder = _TableBuilder(n, lam, partner, table_dtype, dev) if adjacent else None
        host_phi = None
        if builder is not None:
            rows = [min(BLOCK_MODES, r - a0) for a0 in range(0, r, BLOCK_MODES)]
            crc, done = _stream_in(fh, crc, rows, n, torch.complex128,
                                   lambda i, hv: builder.add(i * BLOCK_MODES, hv))
            if not done:
                builder = None              # partner columns are not exact conjugates
        if builder is None:
            # hand-built model (non-conjugate partners): phi goes through the host
            # ReducedModel(phi, ...) constructor path instead
            fh.seek(phi_off)
            crc = crc_head
            host_phi = np.empty((n, r), dtype=np.complex128)
            for a0 in range(0, r, BLOCK_MODES):
                a1 = min(r, a0 + BLOCK_MODES)
                raw = fh.read(16 * n * (a1 - a0))
                crc = zlib.crc32(raw, crc)
                host_phi[:, a0:a1] = np.frombuffer(raw, dtype=_C128).reshape(a1 - a0, n).T
        fh.seek(phi_off + 16 * n * r + 4)
        prov_raw = fh.read(plen)
        crc = zlib.crc32(plen_raw, crc)
        crc = zlib.crc32(prov_raw, crc)
        crc_stored = int(np.frombuffer(fh.read(4), dtype=_U32)[0])
    if crc_stored != crc:
        raise ChecksumError(f"{path}: checksum mismatch (stored {crc_stored:#010x}, computed {crc:#010x})")
    grid_meta = grid_from_kv(kv_loads(grid_raw.decode("utf-8")))
    provenance = kv_loads(prov_raw.decode("utf-8"))
    if builder is None:
        from .modes import modes_from_host_phi
        return ReducedModel(None, lam, sigma, dt, grid_meta, provenance,
                            _modes=modes_from_host_phi(host_phi, lam, dtype=table_dtype, device=dev))
    table, lay = builder.finish()
    return ReducedModel(None, lam, sigma, dt, grid_meta, provenance, _modes=DeviceModes(table, lay))


class _TableBuilder:
    """Decode-table columns (dmd.py:92-120) written into HBM as phi columns
    stream in: self-paired a -> Re phi_a (+ an extra Im column when complex);
    pair a < b -> 2 Re phi_a, -2 Im phi_a, with phi_b checked to be conj(phi_a)."""

    def __init__(self, n, lam, partner, dtype, dev):
        from .modes import TableLayout
        self.n, self.lam, self.partner, self.dev = n, lam, partner, dev
        self.base = TableLayout(lam)                      # columns without extras
        self.col_re = {a: k for k, a in self.base.re_idx}
        self.col_im = {a: k for k, a in self.base.im_idx}
        n_self = sum(1 for a in range(lam.size) if partner[a] == a)
        self.T = alloc_tall(n, self.base.ncol_table + n_self, dtype, "col", device=dev)
        self.extra = []
        self.first = {}

    def add(self, a0, blk: torch.Tensor) -> bool:
        """blk: (b, n) complex128 host rows = phi[:, a0:a0+b].T"""
        t = blk.to(self.dev, non_blocking=False)
        for i in range(blk.shape[0]):
            a = a0 + i
            b = int(self.partner[a])
            col = t[i]
            if b == a:
                self.T.buf[self.col_re[a], : self.n] = col.real.to(self.T.dtype)
                if bool((col.imag != 0).any()):
                    k = self.base.ncol_table + len(self.extra)
                    self.T.buf[k, : self.n] = col.imag.to(self.T.dtype)
                    self.extra.append(a)
            elif b > a:
                self.T.buf[self.col_re[a], : self.n] = (2.0 * col.real).to(self.T.dtype)
                self.T.buf[self.col_im[a], : self.n] = (-2.0 * col.imag).to(self.T.dtype)
                self.first[a] = col.clone()
            else:                                         # b < a: must be the exact conjugate
                ref = self.first.pop(b, None)
                if ref is None or not torch.equal(col, ref.conj()):
                    return False
        return True

    def finish(self):
        from .modes import TableLayout
        lay = TableLayout(self.lam, self.extra)
        return self.T, lay


# ---------------------------------------------------------------------------
# dataset directories (model_io.py:258-336)
# ---------------------------------------------------------------------------
def save_dataset(path, snapshots, density=None):
    """Write a dataset directory from a (device) SnapshotMatrix: snapshots.bin
    is f64 column-major, streamed 8 columns at a time (device transpose +
    pinned D2H) with its CRC32; the manifest as model_io.py:258-294."""
    from .dmd import SnapshotMatrix
    if not isinstance(snapshots, SnapshotMatrix):
        snapshots = SnapshotMatrix(snapshots.states, snapshots.dt, getattr(snapshots, "grid_meta", None),
                                   getattr(snapshots, "meta", None))
    S = snapshots.S
    n, frames = S.n, S.k
    os.makedirs(path, exist_ok=True)
    with open(os.path.join(path, SNAPSHOTS_NAME), "wb") as fh:
        blocks = (S.buf[:n, j0:min(frames, j0 + BLOCK_COLS)].t().to(torch.float64).contiguous()
                  for j0 in range(0, frames, BLOCK_COLS))                  # (cols, n): file order
        crc = _stream_out(fh, 0, blocks, BLOCK_COLS, n, torch.float64)
    grid_kv = grid_to_kv(snapshots.grid_meta)
    manifest = {"kind": "dataset", "grid_kind": grid_kv["kind"]}
    for key, value in grid_kv.items():
        if key != "kind":
            manifest[key] = value
    manifest["dt"] = snapshots.dt
    manifest["frames"] = frames
    manifest["n"] = n
    manifest["layout"] = "u_then_v_row_major"
    manifest["solver"] = snapshots.meta.get("solver", "unknown")
    manifest["snapshots_crc32"] = crc
    manifest["has_density"] = density is not None
    scene = snapshots.meta.get("scene")
    if scene is not None and dataclasses.is_dataclass(scene):
        for f in dataclasses.fields(scene):
            v = getattr(scene, f.name)
            if f.name == "region_disks":
                v = [x for d in v for x in d]
            manifest[f"scene.{f.name}"] = format_value(v)
    elif isinstance(scene, dict):
        for k, v in scene.items():
            manifest[f"scene.{k}"] = format_value(v)
    for key, value in snapshots.meta.items():
        if key in ("scene", "solver"):
            continue
        manifest[f"meta.{key}"] = format_value(value)
    if density is not None:
        density = np.asarray(density, dtype=np.float64)
        dblob = density.reshape(-1, frames).astype(_F64).ravel(order="F").tobytes()
        manifest["density_crc32"] = zlib.crc32(dblob)
        manifest["density_cells"] = density.reshape(-1, frames).shape[0]
        with open(os.path.join(path, DENSITY_NAME), "wb") as fh:
            fh.write(dblob)
    with open(os.path.join(path, MANIFEST_NAME), "w", encoding="utf-8") as fh:
        fh.write(kv_dumps({k: format_value(v) for k, v in manifest.items()}))


def load_dataset(path, device=None, dtype=torch.float64):
    """Read a dataset directory into a device SnapshotMatrix (model_io.py:297-336).
    ``dtype=torch.float32`` keeps the HBM copy in f32 (half the footprint;
    the kernels upcast exactly); the reference keeps f64."""
    from .dmd import SnapshotMatrix
    manifest_path = os.path.join(path, MANIFEST_NAME)
    if not os.path.exists(manifest_path):
        raise SizeMismatchError(f"{path}: missing {MANIFEST_NAME}")
    with open(manifest_path, "r", encoding="utf-8") as fh:
        kv = kv_loads(fh.read())
    if kv.get("kind") != "dataset":
        raise BadMagicError(f"{path}: manifest kind is {kv.get('kind')!r}")
    n, frames = int(kv["n"]), int(kv["frames"])
    snap = os.path.join(path, SNAPSHOTS_NAME)
    size = os.path.getsize(snap)
    if size != 8 * n * frames:
        raise SizeMismatchError(f"{path}: snapshots.bin holds {size} bytes, manifest implies {8 * n * frames}")
    dev = device or dv.default_device()
    S = alloc_tall(n, frames, dtype, "row", device=dev)
    if S.ld > frames:
        S.buf[:, frames:].zero_()
    def put(i, hv):                                                      # (cols, n) host block
        j0 = i * BLOCK_COLS
        S.buf[:n, j0:j0 + hv.shape[0]] = hv.to(dev, non_blocking=False).t().to(dtype)   # device transpose

    with open(snap, "rb") as fh:
        rows = [min(BLOCK_COLS, frames - j0) for j0 in range(0, frames, BLOCK_COLS)]
        crc, _ = _stream_in(fh, 0, rows, n, torch.float64, put)
    if "snapshots_crc32" in kv and crc != int(kv["snapshots_crc32"]):
        raise ChecksumError(f"{path}: snapshots.bin checksum mismatch")
    grid_kv = {"kind": kv.get("grid_kind", "none")}
    for key in ("nx", "ny", "h", "boundary", "solid_cells"):
        if key in kv:
            grid_kv[key] = kv[key]
    meta = {"solver": kv.get("solver", "unknown")}
    scene = {k[len("scene."):]: v for k, v in kv.items() if k.startswith("scene.")}
    if scene:
        meta["scene"] = scene
    for key, value in kv.items():
        if key.startswith("meta."):
            meta[key[len("meta."):]] = value
    return SnapshotMatrix(S, float(kv["dt"]), grid_from_kv(grid_kv), meta)


def load_dataset_density(path):
    """Density frames saved alongside a dataset, or None (model_io.py:339-358)."""
    with open(os.path.join(path, MANIFEST_NAME), "r", encoding="utf-8") as fh:
        kv = kv_loads(fh.read())
    if not parse_bool(kv.get("has_density", "false")):
        return None
    frames, cells = int(kv["frames"]), int(kv["density_cells"])
    with open(os.path.join(path, DENSITY_NAME), "rb") as fh:
        blob = fh.read()
    if len(blob) != 8 * cells * frames:
        raise SizeMismatchError(f"{path}: density.bin size mismatch")
    if "density_crc32" in kv and zlib.crc32(blob) != int(kv["density_crc32"]):
        raise ChecksumError(f"{path}: density.bin checksum mismatch")
    dens = np.frombuffer(blob, dtype=_F64).reshape((cells, frames), order="F").copy()
    if "nx" in kv and "ny" in kv:
        return dens.reshape((int(kv["ny"]), int(kv["nx"]), frames))
    return dens


# ---------------------------------------------------------------------------
# edit spec files (model_io.py:429-466)
# ---------------------------------------------------------------------------
def edit_to_kv(spec):
    return {"kind": "editspec", "r": spec.r, "cluster_threshold": spec.cluster_threshold,
            "weights": spec.weights, "growth_scale": spec.growth_scale, "freq_scale": spec.freq_scale}


def edit_from_kv(kv):
    from .editing import EditSpec
    if kv.get("kind", "editspec") != "editspec":
        raise ValueError("not an edit spec")
    spec = EditSpec(parse_floats(kv["weights"]), parse_floats(kv["growth_scale"]), parse_floats(kv["freq_scale"]),
                    float(kv.get("cluster_threshold", "0.01")))
    if "r" in kv and int(kv["r"]) != spec.r:
        raise ValueError(f"edit spec declares r = {kv['r']} but carries {spec.r} entries")
    return spec


def save_edit(path, spec):
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(kv_dumps({k: format_value(v) for k, v in edit_to_kv(spec).items()}))


def load_edit(path):
    with open(path, "r", encoding="utf-8") as fh:
        return edit_from_kv(kv_loads(fh.read()))


# ---------------------------------------------------------------------------
# scene files (model_io.py:361-422)
# ---------------------------------------------------------------------------
def _scene_fields():
    from .solver import SceneConfig
    return SceneConfig, {f.name: f for f in dataclasses.fields(SceneConfig)}


def scene_to_kv(scene):
    _, fields = _scene_fields()
    out = {}
    for name in fields:
        value = getattr(scene, name)
        if name == "region_disks":
            value = [x for d in value for x in d]
        out[name] = format_value(value)
    return out


def scene_from_kv(kv):
    SceneConfig, fields = _scene_fields()
    kwargs = {}
    for name, fld in fields.items():
        if name not in kv:
            continue
        raw = kv[name]
        if name == "region_disks":
            flat = parse_floats(raw)
            if flat.size % 3:
                raise ValueError("region_disks needs cx,cy,r triples")
            kwargs[name] = tuple(tuple(flat[k:k + 3]) for k in range(0, flat.size, 3))
        elif fld.type in ("int", int):
            kwargs[name] = int(raw)
        elif fld.type in ("float", float):
            kwargs[name] = float(raw)
        elif fld.type in ("bool", bool):
            kwargs[name] = parse_bool(raw)
        elif name == "region_down":
            kwargs[name] = None if raw == "none" else float(raw)
        else:
            kwargs[name] = raw
    return SceneConfig(**kwargs)


def save_scene(path, scene):
    kv = {"kind": "scene"}
    for key, value in scene_to_kv(scene).items():
        kv["scene_kind" if key == "kind" else key] = value
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(kv_dumps(kv))


def load_scene(path):
    with open(path, "r", encoding="utf-8") as fh:
        kv = kv_loads(fh.read())
    if kv.pop("kind", "scene") != "scene":
        raise ValueError(f"{path}: not a scene file")
    if "scene_kind" in kv:
        kv["kind"] = kv.pop("scene_kind")
    return scene_from_kv(kv)
