"""Host-buffer entry points: stream a pinned host batch through the device transforms.

`fwd_inv_host` is what a user with host-resident data calls: the batch is cut
into row chunks; on each of `n_streams` CUDA streams a chunk is copied to the
device, transformed in place by the C-ABI calls (rdfft_fwd, an optional packed
product, rdfft_inv) and copied back, so PCIe host-to-device traffic, device
compute and device-to-host traffic of different chunks overlap.  The device
buffer is caller-provided (no allocation); every transform runs in the CUDA
kernels of librdfft.so.
"""
from __future__ import annotations

import torch

from . import rdfft as R


def fwd_inv_host(xh: torch.Tensor, xd: torch.Tensor, filt: torch.Tensor | None = None, chunk_rows: int = 1 << 16,
                 streams: list | None = None) -> torch.Tensor:
    """In place on the host rows of xh: xh <- IrdFFT(rdFFT(xh) [(.) filt]) through device buffer xd.

    xh: pinned CPU tensor [batch, n]; xd: CUDA tensor of the same shape and dtype (work space owned by
    the caller); filt: optional packed spectrum [1, n] on the device.  Returns xh once the last copy
    back has completed on the streams (the caller synchronises).
    """
    if not xh.is_pinned():
        raise ValueError("xh must be pinned host memory (asynchronous copies)")
    if xd.shape != xh.shape or xd.dtype != xh.dtype or not xd.is_cuda:
        raise ValueError("xd must be a CUDA tensor shaped like xh")
    streams = streams or [torch.cuda.Stream(xd.device) for _ in range(2)]
    cur = torch.cuda.current_stream(xd.device)
    for s in streams:
        s.wait_stream(cur)
    batch = xh.shape[0]
    for i, lo in enumerate(range(0, batch, chunk_rows)):
        hi = min(batch, lo + chunk_rows)
        s = streams[i % len(streams)]
        with torch.cuda.stream(s):
            d = xd[lo:hi]
            d.copy_(xh[lo:hi], non_blocking=True)
            R.rdfft_fwd(d)
            if filt is not None:
                R.rdfft_packed_mul(d, filt)
            R.rdfft_inv(d)
            xh[lo:hi].copy_(d, non_blocking=True)
    for s in streams:
        cur.wait_stream(s)
    return xh
