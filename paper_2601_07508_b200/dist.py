"""Multi-process row partitioner (one process per GPU).

C = A B mod p is split into contiguous row blocks of A / C, one per rank
(``rows_for``); rank ``root`` packs B's words once and NCCL broadcasts them
over NVLink; every rank runs the fused kernel on its rows; the C row blocks
are gathered on ``root`` (grouped NCCL send/recv).  These are the only data
exchanges of the path (north_star: "NCCL over NVLink is used only for that
broadcast and the final gather").

The NCCL communicator lives inside libfpmm_b200.so; torch.distributed (any
backend) only ships the 128-byte NCCL unique id from rank 0 to the others.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

from . import Error, Timing, _check, _dev_ld, _eng, _stream_handle, lib


class Partitioner:
    """Host-side partition logic (pure; usable without a GPU)."""

    def __init__(self, nranks: int, rank: int):
        if nranks < 1 or not 0 <= rank < nranks:
            raise Error("bad rank / world size")
        self.nranks, self.rank = nranks, rank

    def rows_for(self, m: int, u: int, v: int, rank: Optional[int] = None):
        """(row0, rows) of `rank`'s block: ceil(tiles/nranks) GEMM row tiles each."""
        r = self.rank if rank is None else rank
        a, b = C.c_int64(), C.c_int64()
        _check(lib().fpmm_b200_dist_rows(m, self.nranks, r, u, v, C.byref(a), C.byref(b)))
        return a.value, b.value

    @staticmethod
    def chunks_for(rows: int, m: int, k: int, n: int, p: int, u: int, v: int, flags: int = 0):
        """[(start, len)] row chunks of a `rows`-row block: the order in which
        the gathered product computes and ships C to root (fpmm_b200_dist_chunks)."""
        cnt = C.c_int()
        st = (C.c_int64 * 4)()
        ln = (C.c_int64 * 4)()
        _check(lib().fpmm_b200_dist_chunks(m, k, n, p, u, v, flags, rows, C.byref(cnt), st, ln))
        return [(st[i], ln[i]) for i in range(cnt.value)]


_inited = False


def init_from_torch(device: Optional[int] = None) -> Partitioner:
    """Create the library's NCCL communicator for the current torch.distributed group."""
    global _inited
    import torch
    import torch.distributed as td
    rank, world = td.get_rank(), td.get_world_size()
    if device is None:
        device = torch.cuda.current_device()
    n = lib().fpmm_b200_nccl_id_size()
    buf = (C.c_char * n)()
    if rank == 0:
        _check(lib().fpmm_b200_nccl_get_unique_id(C.cast(buf, C.c_void_p)))
    obj = [bytes(buf) if rank == 0 else None]
    td.broadcast_object_list(obj, src=0)
    C.memmove(buf, obj[0], n)
    _check(lib().fpmm_b200_dist_init(C.cast(buf, C.c_void_p), world, rank, device))
    _inited = True
    return Partitioner(world, rank)


def finalize() -> None:
    global _inited
    if _inited:
        _check(lib().fpmm_b200_dist_finalize())
        _inited = False


def mw_product_device(A_rows, B, C_rows, p: int, u: int, v: int, lambda_: int, m: int, *,
                      root: int = 0, C_full=None, stream=None, flags: int = 0,
                      timing: Optional[Timing] = None) -> None:
    """Row-sharded product on device tensors.

    A_rows: this rank's (rows x k) block; B: (k x n) on `root` (ignored
    elsewhere, may be None); C_rows: this rank's (rows x n) output block;
    C_full: optional (m x n) gather target on `root`."""
    k = A_rows.shape[1]
    n = C_rows.shape[1]
    bptr, ldb = (B.data_ptr(), _dev_ld(B)) if B is not None else (None, max(n, 1))
    cf, ldcf = (C_full.data_ptr(), _dev_ld(C_full)) if C_full is not None else (None, max(n, 1))
    sp = _stream_handle(stream, A_rows.device.index)
    _check(lib().fpmm_b200_dist_mw_product_device(
        A_rows.data_ptr(), max(k, 1) if A_rows.shape[0] <= 1 else _dev_ld(A_rows), bptr, ldb,
        C_rows.data_ptr(), max(n, 1) if C_rows.shape[0] <= 1 else _dev_ld(C_rows), cf, ldcf, m, k, n,
        p, u, v, lambda_, root, sp, _eng(flags), C.byref(timing) if timing is not None else None))


def mw_product_host(A_rows_host, B_host, C_host, p: int, u: int, v: int, lambda_: int, m: int, *,
                    root: int = 0, scratch=None, timing: Optional[Timing] = None, flags: int = 0):
    """Host-buffer (pinned numpy / torch CPU) variant of `mw_product_device`:
    H2D of this rank's A rows (and B on root), the sharded product, C gathered
    on root and copied back into C_host.  `scratch` caches device buffers."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    a = torch.as_tensor(A_rows_host)
    sc = scratch if scratch is not None else {}

    def buf(name, shape):
        t = sc.get(name)
        if t is None or tuple(t.shape) != tuple(shape):
            t = torch.empty(shape, dtype=torch.float64, device=dev)
            sc[name] = t
        return t

    dA = buf("A", a.shape)
    dA.copy_(a, non_blocking=True)
    n = None
    dB = None
    if B_host is not None:
        b = torch.as_tensor(B_host)
        dB = buf("B", b.shape)
        dB.copy_(b, non_blocking=True)
        n = b.shape[1]
    if n is None:
        n = C_host.shape[1] if C_host is not None else sc.get("n")
    if n is None:
        raise Error("non-root ranks must know n (pass scratch={'n': n})")
    dC = buf("Crows", (a.shape[0], n))
    dCf = buf("Cfull", (m, n)) if C_host is not None else None
    # the product runs on the stream that carries the H2D copies above (torch's
    # current stream), so the packers never read A or B before they land
    mw_product_device(dA, dB, dC, p, u, v, lambda_, m, root=root, C_full=dCf, timing=timing,
                      flags=flags, stream=torch.cuda.current_stream())
    if C_host is not None:
        torch.as_tensor(C_host).copy_(dCf)
    torch.cuda.synchronize()
