"""Host <-> device conversion for the reference-compatible list API.

Keys and values travel as integer tensors holding the table's storage bit
pattern (int32 for <= 32-bit fields, int64 otherwise; uint64 keys >= 2^63
simply appear negative in the int64 view).  CUDA tensors are used in place;
Python sequences and numpy arrays are staged through pinned host memory.
"""
from __future__ import annotations

import numpy as np
import torch


def torch_dtype(bits: int) -> torch.dtype:
    return torch.int32 if bits <= 32 else torch.int64


def np_dtype(bits: int):
    return np.uint32 if bits <= 32 else np.uint64


def _np_signed(bits: int):
    return np.int32 if bits <= 32 else np.int64


def to_numpy(seq, bits: int, what: str = "key") -> np.ndarray:
    """Python ints / arrays -> contiguous unsigned array of the storage width."""
    if isinstance(seq, np.ndarray):
        arr = seq
        if arr.dtype.kind == "i" and arr.size and arr.min() < 0:
            raise ValueError(f"negative {what}")
        arr = arr.astype(np.uint64, copy=False)
    else:
        seq = list(seq)
        try:
            arr = np.array(seq, dtype=np.uint64) if seq else np.empty(0, dtype=np.uint64)
        except (OverflowError, ValueError, TypeError) as err:
            raise ValueError(f"{what}s must be integers in [0, 2^64)") from err
    if bits <= 32:
        if arr.size and arr.max() > np.uint64(0xFFFFFFFF):
            raise ValueError(f"{what} does not fit in {bits} bits")
        arr = arr.astype(np.uint32)
    return np.ascontiguousarray(arr)


def to_device(x, bits: int, device: int, what: str = "key") -> torch.Tensor:
    """Anything array-like -> contiguous CUDA tensor of the storage width."""
    dt = torch_dtype(bits)
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == dt and x.is_contiguous() and x.device.index == device:
            return x
        if x.dtype in (torch.int32, torch.int64, torch.uint32, torch.uint64) and x.element_size() == \
                torch.tensor([], dtype=dt).element_size():
            return x.contiguous().view(dt).to(f"cuda:{device}", non_blocking=True)
        x = x.cpu().numpy()
    arr = to_numpy(x, bits, what)
    host = torch.from_numpy(arr.view(_np_signed(bits)))
    if host.numel() > (1 << 16):
        host = host.pin_memory()
    return host.to(f"cuda:{device}", non_blocking=True)


def from_device(t: torch.Tensor, bits: int) -> np.ndarray:
    """CUDA integer tensor -> unsigned numpy array (bit-exact)."""
    a = t.cpu().numpy()
    return a.view(np.uint32 if a.dtype.itemsize == 4 else np.uint64)


def stream_of(device: int, stream=None) -> int:
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def split_pairs(pairs) -> tuple[list, list]:
    pairs = list(pairs)
    return [k for k, _ in pairs], [v for _, v in pairs]


class Staging:
    """Persistent device staging buffers of one table's host-buffer pipeline (three chunk
    slots per input stream), with an event per slot marking when its last op consumed it.

    Reusing them across calls removes the whole-stream wait a freshly allocated buffer
    needs: the next call's H2D copies wait only for the slot they overwrite, so the
    copies of a retrieve_host overlap the kernels still running for the insert_host
    issued before it."""

    NB = 3

    def __init__(self):
        self._sets = {}

    def get(self, device: int, chunk: int, dtypes: tuple):
        key = (device, chunk, dtypes)
        st = self._sets.get(key)
        if st is None:
            dev = torch.device("cuda", device)
            bufs = [[torch.empty(chunk, dtype=dt, device=dev) for dt in dtypes] for _ in range(self.NB)]
            free = [None] * self.NB
            s_in = torch.cuda.Stream(dev)
            s_in.wait_stream(torch.cuda.current_stream(dev))  # fresh memory: after its previous users
            st = self._sets[key] = (bufs, free, s_in, torch.cuda.Stream(dev))
        return st


def pipelined(device: int, inputs: list, outputs: list, run, chunk: int, staging: Staging | None = None) -> None:
    """Stream host inputs through a device op in chunks: H2D copies, kernels and D2H
    copies of consecutive chunks overlap on three CUDA streams.

    inputs / outputs: equal-length pinned host tensors (outputs are filled in place).
    run(list_of_device_input_slices, stream) -> list of device outputs, one per output.
    The caller's current stream waits for the whole pipeline (the D2H copies included)
    when this returns; the host does not (callers synchronise when they need the data).
    """
    n = inputs[0].numel()
    if n == 0:
        return
    dev = torch.device("cuda", device)
    compute = torch.cuda.current_stream(dev)
    if staging is not None:
        bufs, free, s_in, s_out = staging.get(device, min(chunk, n), tuple(x.dtype for x in inputs))
    else:
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        bufs = [[torch.empty(min(chunk, n), dtype=x.dtype, device=dev) for x in inputs] for _ in range(3)]
        free = [None] * 3
        s_in.wait_stream(compute)   # fresh buffers: order after whatever last used the memory
    nb = len(bufs)
    for c, lo in enumerate(range(0, n, chunk)):
        hi = min(n, lo + chunk)
        m = hi - lo
        b = c % nb
        ev_in = torch.cuda.Event()
        with torch.cuda.stream(s_in):
            if free[b] is not None:
                s_in.wait_event(free[b])
            for d, x in zip(bufs[b], inputs):
                d[:m].copy_(x[lo:hi], non_blocking=True)
            ev_in.record(s_in)
        compute.wait_event(ev_in)
        outs = run([d[:m] for d in bufs[b]], compute)
        ev_done = torch.cuda.Event()
        ev_done.record(compute)
        free[b] = ev_done  # the inputs are consumed once the op has run: the next H2D into
        with torch.cuda.stream(s_out):  # this buffer need not wait for the D2H below
            s_out.wait_event(ev_done)
            for o, y in zip(outs, outputs):
                o.record_stream(s_out)
                y[lo:hi].copy_(o, non_blocking=True)
    compute.wait_stream(s_out)
    if staging is None:
        for bb in bufs:
            for d in bb:
                d.record_stream(s_in)
