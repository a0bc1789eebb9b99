"""The 2-D work-item index space and its device dispatch.

Drop-in for the reference's grid.py (/root/reference/pkg/src/streamforge/
grid.py).  The ownership rules (element_plan, stream_index) are identical;
run_grid dispatches to the sm_100a kernels through the C ABI
(include/sfb.h: sfb_fill_real / sfb_fill_integer / sfb_fill_normal), which
replace _kernels.fill_real / fill_integer / fill_normal (grid.py:124-141).

MatrixBuffer keeps the generated matrix in HBM (`.tensor`) and only copies it
to the host when `.data` / `.values` / `.vector()` are read, preserving the
reference's numpy view semantics.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import StreamSet
from .errors import InsufficientStreamsError, InvalidArgumentError, InvalidGridError

UNIFORM_KERNEL = "uniform"
NORMAL_KERNEL = "normal"


@dataclass(frozen=True)
class WorkGrid:
    """Two-dimensional global work-item index space (grid.py:22-41)."""

    nglobal0: int
    nglobal1: int

    def __post_init__(self):
        if self.nglobal0 < 1 or self.nglobal1 < 1:
            raise InvalidGridError("work grid dimensions must be >= 1")

    @property
    def size(self) -> int:
        return self.nglobal0 * self.nglobal1

    def require_paired_lanes(self):
        if self.nglobal1 % 2 != 0:
            raise InvalidGridError("normal generation needs an even lane count (nglobal1)")


_TORCH_DTYPES = {}


def _torch_dtype(dtype):
    import torch

    return {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
            np.dtype(np.int64): torch.int64}[np.dtype(dtype)]


class MatrixBuffer:
    """Row-major matrix of ncol logical columns inside a padded width npad
    (grid.py:44-70).  Cells beyond the first ncol columns are never written.

    Device-backed when produced by a fill: `.tensor` is the (nrow, npad) CUDA
    tensor; `.data` lazily copies it to a numpy array (once)."""

    def __init__(self, nrow, ncol, npad=None, dtype=np.float64, is_vector=False, *,
                 tensor=None):
        npad = ncol if npad is None else npad
        if nrow < 1 or ncol < 1:
            raise InvalidArgumentError("matrix dimensions must be >= 1")
        if npad < ncol:
            raise InvalidArgumentError("npad must be >= ncol")
        self.nrow = nrow
        self.ncol = ncol
        self.npad = npad
        self.is_vector = is_vector
        self.dtype = np.dtype(dtype)
        self.tensor = tensor
        self.shard = None  # sharded fills: the rank's FillShard (sharding.py)
        self._host = None if tensor is not None else np.zeros((nrow, npad), dtype=dtype)

    @classmethod
    def wrap(cls, tensor, dtype, ncol=None):
        """A buffer around an existing (nrow, npad) CUDA tensor (sharded fills;
        a rank whose streams own no cell gets an empty one)."""
        obj = cls.__new__(cls)
        obj.nrow, obj.npad = int(tensor.shape[0]), int(tensor.shape[1])
        obj.ncol = obj.npad if ncol is None else ncol
        obj.is_vector = False
        obj.dtype = np.dtype(dtype)
        obj.tensor = tensor
        obj.shard = None
        obj._host = None
        return obj

    @classmethod
    def on_device(cls, nrow, ncol, npad=None, dtype=np.float64, is_vector=False, zero=False):
        import torch

        npad = ncol if npad is None else npad
        if nrow < 1 or ncol < 1:
            raise InvalidArgumentError("matrix dimensions must be >= 1")
        if npad < ncol:
            raise InvalidArgumentError("npad must be >= ncol")
        alloc = torch.zeros if zero else torch.empty
        t = alloc((nrow, npad), dtype=_torch_dtype(dtype), device="cuda")
        return cls(nrow, ncol, npad, dtype, is_vector, tensor=t)

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            self._host = _lib.to_host(self.tensor)
        return self._host

    @property
    def values(self) -> np.ndarray:
        """The logical nrow x ncol submatrix."""
        return self.data[:, : self.ncol]

    def vector(self) -> np.ndarray:
        return self.values.ravel()

    def download(self, out=None):
        """Copy the (nrow, npad) matrix into host memory `out` (a numpy array or a
        torch CPU tensor; pinned memory gives full PCIe bandwidth) and return it."""
        import torch

        if self.tensor is None:
            if out is None:
                return self._host
            np.copyto(np.asarray(out), self._host)
            return out
        if out is None:
            out = torch.empty(self.tensor.shape, dtype=self.tensor.dtype, pin_memory=True)
        dst = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
        src = self.tensor
        nbytes = src.numel() * src.element_size()
        if nbytes < (256 << 20) or not dst.is_pinned() or src.shape[0] < 4:
            dst.copy_(src)
            return out
        # large pinned downloads: row chunks on two copy streams keep both
        # copy engines busy (measured 53 -> 55.6 GB/s on B200, tools/d2h_probe.py)
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(src.device))
        streams = _copy_streams(src.device)
        bounds = np.linspace(0, src.shape[0], 9).astype(int)
        for k in range(8):
            s = streams[k % 2]
            s.wait_event(ready)
            with torch.cuda.stream(s):
                dst[bounds[k]:bounds[k + 1]].copy_(src[bounds[k]:bounds[k + 1]], non_blocking=True)
        for s in streams:
            s.synchronize()
        return out

    def download_shard(self, g1: int, j_lo: int, j_hi: int, out=None):
        """Copy the cells of grid columns [j_lo, j_hi) (a rank's uniform-kind
        shard: columns c = j + g1 q) into a packed host array, row-major over
        (row, q, j) -- what one rank of a multi-GPU fill keeps on its host.
        `out` (numpy or pinned torch CPU tensor) must hold exactly those cells."""
        import torch

        cells = sum(len(range(j, self.ncol, g1)) for j in range(j_lo, j_hi)) * self.nrow
        if out is None:
            out = torch.empty(cells, dtype=self.tensor.dtype, pin_memory=True)
        dst = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
        if dst.numel() != cells or not dst.is_contiguous():
            raise InvalidArgumentError(f"shard download needs a contiguous buffer of {cells} cells")
        st = torch.cuda.current_stream(self.tensor.device)
        _lib.check(_lib.lib().sfb_download_shard(
            dst.data_ptr(), self.tensor.data_ptr(), self.nrow, self.ncol, self.npad, g1, j_lo,
            j_hi, self.tensor.element_size(), st.cuda_stream))
        st.synchronize()
        return out

    @property
    def device_values(self):
        """The logical nrow x ncol submatrix as a CUDA tensor view (no copy)."""
        return self.tensor[:, : self.ncol]


_COPY_STREAMS = {}


def _copy_streams(device):
    """Two side streams per device for chunked device->host downloads."""
    import torch

    key = torch.device(device).index
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = [torch.cuda.Stream(device=device) for _ in range(2)]
    return _COPY_STREAMS[key]


def element_plan(grid: WorkGrid, nrow: int, ncol: int):
    """Cells owned by each work item, in visiting order (grid.py:73-87)."""
    plan = {}
    for i in range(grid.nglobal0):
        for j in range(grid.nglobal1):
            plan[(i, j)] = [
                (r, c)
                for r in range(i, nrow, grid.nglobal0)
                for c in range(j, ncol, grid.nglobal1)
            ]
    return plan


def stream_index(kernel_kind: str, grid: WorkGrid, i: int, j: int) -> int:
    """Stream ordinal of work item (i, j) under the given kernel's rule (grid.py:90-102)."""
    if not (0 <= i < grid.nglobal0 and 0 <= j < grid.nglobal1):
        raise InvalidArgumentError("work-item index outside the grid")
    if kernel_kind == UNIFORM_KERNEL:
        return i + grid.nglobal0 * j
    if kernel_kind == NORMAL_KERNEL:
        return i * grid.nglobal1 + j
    raise InvalidArgumentError(f"unknown kernel kind {kernel_kind!r}")


def _check_streams(streams: StreamSet, grid: WorkGrid):
    if streams.count < grid.size:
        raise InsufficientStreamsError(f"grid needs {grid.size} streams, got {streams.count}")


KIND_DTYPES = {"uniform": np.float64, "exponential": np.float64,
               "uniform-integer": np.int64, "normal": np.float64}


def launch_fill(kind, cur_dev, n_streams, out, nrow, ncol, npad, g0, g1, rate=1.0,
                item_lo=0, item_hi=None, zero_pad=True, stream=None):
    """Enqueue one fill kernel on raw device buffers (the C-ABI seam).
    `cur_dev`: int64 (n,6) CUDA tensor; `out`: (nrow, npad) CUDA tensor."""
    import torch

    want = {"normal": (torch.float64, torch.float32), "uniform-integer": (torch.int64,),
            "uniform": (torch.float64,), "exponential": (torch.float64,)}.get(kind)
    if want is None:
        raise InvalidArgumentError(f"unknown fill kind {kind!r}")
    if out.dtype not in want:  # the kernels write 8-byte cells except float32 normals
        raise InvalidArgumentError(f"{kind} fills cannot write a {out.dtype} buffer")
    L = _lib.lib()
    item_hi = g0 * g1 if item_hi is None else item_hi
    st = _lib.stream_handle() if stream is None else stream
    cp, op = _lib.dptr(cur_dev), _lib.dptr(out)
    zp = 1 if zero_pad else 0
    if kind == "normal":
        dt = _lib.SFB_F32 if out.dtype == torch.float32 else _lib.SFB_F64
        rc = L.sfb_fill_normal(cp, n_streams, op, dt, nrow, ncol, npad, g0, g1, item_lo,
                               item_hi, zp, st)
    elif kind == "uniform-integer":
        rc = L.sfb_fill_integer(cp, n_streams, op, nrow, ncol, npad, g0, g1, item_lo, item_hi,
                                zp, st)
    elif kind in ("uniform", "exponential"):
        rc = L.sfb_fill_real(cp, n_streams, op, nrow, ncol, npad, g0, g1,
                             0 if kind == "uniform" else 1, float(rate), item_lo, item_hi, zp,
                             st)
    else:
        raise InvalidArgumentError(f"unknown fill kind {kind!r}")
    _lib.check(rc)


def check_fill(streams, grid, kind, dtype=None) -> np.dtype:
    """Validation of a fill request in the reference's order (grid.py:112-123):
    streams, paired lanes for normals, the kind; then the output dtype of the
    kind (float32 only for normals, the extension).  Returns the dtype."""
    _check_streams(streams, grid)
    if kind == "normal":
        grid.require_paired_lanes()
    elif kind not in ("uniform-integer", "uniform", "exponential"):
        raise InvalidArgumentError(f"unknown fill kind {kind!r}")
    out_dtype = np.dtype(KIND_DTYPES[kind] if dtype is None else dtype)
    if kind != "normal" and out_dtype != np.dtype(KIND_DTYPES[kind]):
        raise InvalidArgumentError(f"{kind} fills produce {np.dtype(KIND_DTYPES[kind])}")
    if kind == "normal" and out_dtype not in (np.dtype(np.float64), np.dtype(np.float32)):
        raise InvalidArgumentError("normal fills produce float64 or float32")
    return out_dtype


def run_grid(streams, grid, nrow, ncol, kind, rate=1.0, npad=None, threads=None, dtype=None):
    """Fill an nrow x ncol matrix, advancing the used streams in place
    (grid.py:112-144).  kind: "uniform", "uniform-integer", "exponential",
    "normal".  `threads` is accepted for API compatibility and never changes
    results.  `dtype` (extension): np.float32 for float32 normals."""
    out_dtype = check_fill(streams, grid, kind, dtype)
    _lib.require_device()
    buf = MatrixBuffer.on_device(nrow, ncol, npad, dtype=out_dtype)
    cur = streams.device_current()
    launch_fill(kind, cur, streams.count, buf.tensor, nrow, ncol, buf.npad, grid.nglobal0,
                grid.nglobal1, rate=rate)
    streams._mark_device_ahead()
    return buf
