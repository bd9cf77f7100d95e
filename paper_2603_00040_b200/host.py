"""Host-buffer entry points: H2D, compute and D2H overlapped across head chunks.

The reference API is host-memory in, host-memory out (flash.py:176, 249, 317
take and return NumPy arrays). Every (batch, head) pair is independent
(oracle.py:96-103), so a batched call splits the heads into chunks and runs a
three-stage pipeline on three CUDA streams:

    h2d stream      copy chunk c+1 inputs   (pinned host -> HBM input slot)
    compute stream  kernels of chunk c      (the caller's current stream)
    d2h stream      copy chunk c-1 outputs  (HBM output slot -> host buffers)

Upload and download use the two PCIe directions concurrently and both hide the
kernels, so a call costs about max(H2D, D2H, compute) plus one chunk of each
instead of their sum. All device memory is owned by a per-device
``HostPipeline``: two input slots, two output slots and two kernel workspaces,
allocated once and recycled under events (no allocator traffic per chunk, no
host synchronisation inside or between calls). By default the call returns
once the host outputs are complete (host memory in, host memory out, like the
reference); with ``sync=False`` it returns once the last download is queued
and the caller's current stream is made to wait for it.
"""

from __future__ import annotations

import threading

import torch

_PIPES = {}
_LOCK = threading.Lock()


class HostPipeline:
    """Per-device streams, slot buffers and the events that recycle them."""

    def __init__(self, device):
        self.device = device
        self.h2d = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)
        self.bufs = {}                  # name -> [slot0, slot1]
        self.in_free = [None, None]     # compute finished reading input slot s
        self.out_free = [None, None]    # download finished reading output slot s
        self.lock = threading.Lock()    # one pipelined call at a time per device (shared slots)

    def slots(self, name, shape, dtype):
        """Two device buffers of at least ``shape``; reallocated (after a device
        sync, so no in-flight work still uses the old ones) when too small."""
        cur = self.bufs.get(name)
        need = 1
        for s in shape:
            need *= int(s)
        if cur is None or cur[0].dtype != dtype or cur[0].numel() < need:
            if cur is not None:
                torch.cuda.synchronize(self.device)
            cur = [torch.empty(need, dtype=dtype, device=self.device) for _ in range(2)]
            self.bufs[name] = cur
        return [b[:need].view(shape) for b in cur]


def pipeline(device=None):
    device = device or torch.device("cuda", torch.cuda.current_device())
    key = device.index if device.index is not None else torch.cuda.current_device()
    with _LOCK:
        if key not in _PIPES:
            _PIPES[key] = HostPipeline(torch.device("cuda", key))
        return _PIPES[key]


def _pinned(t):
    return t if t.is_pinned() else t.pin_memory()


def run_pipelined(fn, host_inputs, host_outputs, chunk_heads, scratch=(), device=None, sync=True):
    """Run ``fn`` over head chunks of host tensors with overlapped transfers.

    host_inputs:  CPU tensors whose dim 0 is the head index (same length H).
    host_outputs: CPU tensors (pinned for real overlap) with dim 0 = H; filled
                  in place.
    scratch:      (name, per-chunk shape or callable(heads) -> shape, dtype)
                  device buffers fn needs per chunk (e.g. kernel workspaces),
                  double-buffered like the slots.
    fn(dev_inputs, dev_outputs, dev_scratch) writes chunk results into
                  dev_outputs (views shaped like host_output[lo:hi]).
    sync:         wait for the last download before returning, so the host
                  outputs can be read at once (the reference contract). With
                  sync=False the caller's current stream is only made to wait
                  for it: read the outputs after synchronising that stream.
    """
    heads = host_inputs[0].shape[0]
    if any(t.shape[0] != heads for t in list(host_inputs) + list(host_outputs)):
        raise ValueError("all host buffers need the same leading (head) dimension")
    pipe = pipeline(device)
    with pipe.lock:
        _run(pipe, fn, host_inputs, host_outputs, heads, chunk_heads, scratch)
    if sync:
        torch.cuda.current_stream(pipe.device).synchronize()


def _run(pipe, fn, host_inputs, host_outputs, heads, chunk_heads, scratch):
    chunk_heads = max(1, min(int(chunk_heads), heads))
    host_inputs = [_pinned(t.contiguous()) for t in host_inputs]
    comp = torch.cuda.current_stream(pipe.device)
    h2d, d2h = pipe.h2d, pipe.d2h
    # the pipeline starts after everything already queued on the caller's stream
    h2d.wait_stream(comp)
    d2h.wait_stream(comp)
    ins = [pipe.slots(f"in{i}", (chunk_heads,) + tuple(t.shape[1:]), t.dtype) for i, t in enumerate(host_inputs)]
    outs = [pipe.slots(f"out{i}", (chunk_heads,) + tuple(t.shape[1:]), t.dtype) for i, t in enumerate(host_outputs)]
    scr = []
    for name, shape, dtype in scratch:
        shp = shape(chunk_heads) if callable(shape) else shape
        scr.append(pipe.slots(f"scratch_{name}", tuple(shp), dtype))
    for c, (lo, hi) in enumerate(_chunks(heads, chunk_heads)):
        n = hi - lo
        s = c % 2
        if pipe.in_free[s] is not None:
            h2d.wait_event(pipe.in_free[s])
        with torch.cuda.stream(h2d):
            dev_in = []
            for buf, t in zip(ins, host_inputs):
                dst = buf[s][:n]
                dst.copy_(t[lo:hi], non_blocking=True)
                dev_in.append(dst)
        loaded = torch.cuda.Event()
        loaded.record(h2d)
        comp.wait_event(loaded)
        if pipe.out_free[s] is not None:
            comp.wait_event(pipe.out_free[s])
        dev_out = [buf[s][:n] for buf in outs]
        with torch.cuda.stream(comp):
            fn(dev_in, dev_out, [b[s] for b in scr])
        done = torch.cuda.Event()
        done.record(comp)
        pipe.in_free[s] = done
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            for o, h in zip(dev_out, host_outputs):
                h[lo:hi].copy_(o, non_blocking=True)
        fetched = torch.cuda.Event()
        fetched.record(d2h)
        pipe.out_free[s] = fetched
    comp.wait_stream(d2h)
    comp.wait_stream(h2d)


def _chunks(heads, chunk):
    """[lo, hi) head ranges: full chunks, with the last full chunk cut into
    quarters -- only the final chunk's kernels and download are not hidden
    behind an upload, so a short tail shortens the exposed end."""
    bounds = list(range(0, heads, chunk)) + [heads]
    spans = [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1)]
    if len(spans) > 1 and chunk >= 4:
        lo, hi = spans.pop()
        step = max(1, -(-(hi - lo) // 4))
        spans += [(a, min(hi, a + step)) for a in range(lo, hi, step)]
    return spans


def default_chunk(heads, per_head_bytes, items_per_head=None, sms=None):
    """Heads per chunk: ~16 chunks (the first upload and the last download are
    not overlapped, so smaller chunks shorten the exposed ends), at least 16 MB
    per chunk so the copies stay near the PCIe rate, and -- when the kernels
    are persistent over (head, 128-row tile) items -- at least ~8 waves of
    items per chunk so a compute-heavy chunk does not end in a mostly idle
    wave."""
    target = max(1, heads // 16)
    min_heads = max(1, (16 << 20) // max(1, per_head_bytes))
    if items_per_head:
        if sms is None:
            sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        min_heads = max(min_heads, -(-8 * sms // items_per_head))
    return min(heads, max(target, min_heads))
