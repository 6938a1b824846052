"""Host-resident batches through the kernels with the PCIe copies overlapped.

`run_pipelined(fn, h_in, h_out, chunks)` splits a pinned host batch [count, ...] into chunks
and cycles them over `nstreams` CUDA streams: the H2D copy of chunk i+1, the kernel of
chunk i and the D2H copy of chunk i-1 run concurrently (PCIe is full duplex), so a
host-to-host call approaches max(H2D, D2H) time instead of their sum.  `fn(d_in, d_out,
stream, lo)` is any batched entry point (e.g. dmm.partition_general with out=, stream=);
`lo` is the chunk's first instance index.
"""
from __future__ import annotations

import torch


class DeviceSlots:
    """Reusable device buffers per stream slot (allocation stays out of the steady state)."""

    def __init__(self, chunk_shape, dtype, nstreams: int, device="cuda"):
        self.streams = [torch.cuda.Stream(device=device) for _ in range(nstreams)]
        self.din = [torch.empty(chunk_shape, dtype=dtype, device=device) for _ in range(nstreams)]
        self.dout = [torch.empty(chunk_shape, dtype=dtype, device=device) for _ in range(nstreams)]


def run_pipelined(fn, h_in: torch.Tensor, h_out: torch.Tensor, chunks: int = 8, nstreams: int = 3,
                  slots: DeviceSlots | None = None) -> DeviceSlots:
    count = h_in.shape[0]
    per = (count + chunks - 1) // chunks
    if slots is None:
        slots = DeviceSlots((per,) + tuple(h_in.shape[1:]), h_in.dtype, nstreams)
    cur = torch.cuda.current_stream()
    done = []
    for i in range(chunks):
        lo, hi = i * per, min(count, (i + 1) * per)
        if lo >= hi:
            break
        k = i % len(slots.streams)
        s = slots.streams[k]
        s.wait_stream(cur) if i < len(slots.streams) else None
        with torch.cuda.stream(s):
            din = slots.din[k][: hi - lo]
            dout = slots.dout[k][: hi - lo]
            din.copy_(h_in[lo:hi], non_blocking=True)
            fn(din, dout, s, lo)
            h_out[lo:hi].copy_(dout, non_blocking=True)
        done.append(s)
    for s in slots.streams:
        cur.wait_stream(s)
    return slots
