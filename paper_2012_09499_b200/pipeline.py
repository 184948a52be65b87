"""End-to-end host -> device -> host pipeline over frame chunks.

``ChunkedRunner`` splits a batch of F frames into chunks, each with its own
graph-captured step (``CapturedStep``), and runs chunk c's host->device copy,
compute and device->host copy on three CUDA streams, so the copy engines
overlap compute of the neighbouring chunks (the maps' device->host transfer
of the C2 workload, 62 MB, is the longest leg).  Cross-call dependencies
keep a chunk's static buffers from being overwritten while the previous call
still reads them.
"""

from __future__ import annotations

import torch

from . import _native as N
from .plan import CapturedStep

MIN_CHUNK_FRAMES = 32  # one tensor-core frame tile


def chunk_bounds(F: int, chunks: int = 4, sizes=None):
    """[lo, hi) frame ranges: ``chunks`` balanced chunks of >= 32 frames, or
    explicit chunk ``sizes`` (the last absorbs any remainder; e.g. multiples
    of the 160-frame tensor-core tile with a short last chunk, whose maps
    leave the device last)."""
    if sizes is not None:
        out, lo = [], 0
        for n in sizes:
            if lo >= F:
                break
            hi = min(F, lo + int(n))
            out.append((lo, hi))
            lo = hi
        if lo < F:
            out[-1] = (out[-1][0], F) if out else (0, F)
        return out
    chunks = max(1, min(chunks, F // MIN_CHUNK_FRAMES or 1))
    base, rem = divmod(F, chunks)
    out, lo = [], 0
    for c in range(chunks):
        hi = lo + base + (1 if c < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


class ChunkedRunner:
    """Pipelined ``plan.run`` over host buffers (pinned for async copies)."""

    def __init__(self, plan, F, M=None, path="approx", chunks=4, maps=True, weighting="phat",
                 phat_floor=None, audio=None, sizes=None):
        """``audio=(frame_length, hop_length, window)``: inputs are [M, L]
        audio (F = its frame count); each chunk's graph runs K0 on the chunk's
        sample span (spans of neighbouring chunks overlap by N - hop)."""
        self.plan, self.F, self.path, self.want_maps = plan, F, path, maps
        self.bounds = chunk_bounds(F, chunks, sizes)
        dev = plan.device
        M = M if M is not None else plan.M
        self.audio = None
        if audio is not None:
            n, hop, window = audio
            hop = n // 2 if hop is None else int(hop)
            self.audio = (n, hop, window)
            self.spans = [(lo * hop, (hi - 1) * hop + n) for lo, hi in self.bounds]
            self.steps = [CapturedStep(plan, hi - lo, M, path, maps, weighting, phat_floor,
                                       audio=(b - a, n, hop, window))
                          for (lo, hi), (a, b) in zip(self.bounds, self.spans)]
        else:
            self.steps = [CapturedStep(plan, hi - lo, M, path, maps, weighting, phat_floor)
                          for lo, hi in self.bounds]
        self.s_in = torch.cuda.Stream(dev)
        self.s_comp = torch.cuda.Stream(dev)
        self.s_out = torch.cuda.Stream(dev)
        n = len(self.bounds)
        self.ev_in = [torch.cuda.Event() for _ in range(n)]
        self.ev_comp = [torch.cuda.Event() for _ in range(n)]
        self.ev_out = [torch.cuda.Event() for _ in range(n)]
        self._first = True

    @property
    def launches(self):
        """Kernels per call (all chunks)."""
        return sum(s.launches for s in self.steps)

    def run(self, Y_host, maps_host=None, argmax_host=None):
        """Enqueue one pass: Y_host [F, M, Kb] complex64 (or [M, L] float32
        audio) in pinned memory -> maps_host [F, J] float32 and argmax_host
        [F] int32 (pinned).  Asynchronous with respect to the host; the
        caller's current stream waits for the last device->host copy, and
        the first host->device copy waits for the caller's prior work."""
        self._check_host(Y_host, maps_host, argmax_host)
        self.s_in.wait_stream(torch.cuda.current_stream(self.plan.device))
        for c, (lo, hi) in enumerate(self.bounds):
            st = self.steps[c]
            with torch.cuda.stream(self.s_in):
                if not self._first:  # previous call's compute has read the input
                    self.s_in.wait_event(self.ev_comp[c])
                if self.audio is not None:
                    # the chunk's sample span of every channel: one strided
                    # DMA (a column block of the host [M, L] array)
                    a, b = self.spans[c]
                    M = st.x.shape[0]
                    es = Y_host.element_size()
                    N.call("srpb_copy_rows_h2d", N.ptr(st.x), st.x.stride(0) * es,
                           Y_host.data_ptr() + a * es, Y_host.stride(0) * es, (b - a) * es, M,
                           self.s_in.cuda_stream)
                else:
                    st.Y.copy_(Y_host[lo:hi], non_blocking=True)
                self.ev_in[c].record(self.s_in)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(self.ev_in[c])
                if not self._first:  # previous call's copy-out has read the outputs
                    self.s_comp.wait_event(self.ev_out[c])
                st.graph.replay()
                self.ev_comp[c].record(self.s_comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_comp[c])
                if maps_host is not None and st.maps is not None:
                    maps_host[lo:hi].copy_(st.maps, non_blocking=True)
                if argmax_host is not None:
                    argmax_host[lo:hi].copy_(st.argmax, non_blocking=True)
                self.ev_out[c].record(self.s_out)
        self._first = False
        torch.cuda.current_stream(self.plan.device).wait_stream(self.s_out)


    def _check_host(self, Y_host, maps_host, argmax_host):
        """Host buffers the DMA engines read and write must be CPU tensors
        covering every chunk (the audio path copies with raw pointers)."""
        for name, t in (("input", Y_host), ("maps_host", maps_host),
                        ("argmax_host", argmax_host)):
            if t is not None and (not isinstance(t, torch.Tensor) or t.device.type != "cpu"):
                raise ValueError(f"{name} must be a CPU (pinned) tensor")
        st = self.steps[0]
        if self.audio is not None:
            if (Y_host.dim() != 2 or Y_host.dtype != torch.float32 or Y_host.stride(1) != 1
                    or Y_host.shape[0] != st.x.shape[0] or Y_host.shape[1] < self.spans[-1][1]):
                raise ValueError(f"audio must be a row-major float32 [M={st.x.shape[0]}, "
                                 f">= {self.spans[-1][1]}] host array, got "
                                 f"{Y_host.dtype} {tuple(Y_host.shape)}")
        elif (Y_host.dim() != 3 or Y_host.shape[0] < self.F
              or tuple(Y_host.shape[1:]) != tuple(st.Y.shape[1:])):
            raise ValueError(f"Y must be [>= {self.F}, {st.Y.shape[1]}, {st.Y.shape[2]}], got "
                             f"{tuple(Y_host.shape)}")
        if maps_host is not None and (maps_host.dim() != 2 or maps_host.shape[0] < self.F
                                      or maps_host.shape[1] != self.plan.J):
            raise ValueError(f"maps_host must be [>= {self.F}, {self.plan.J}]")
        if argmax_host is not None and argmax_host.numel() < self.F:
            raise ValueError(f"argmax_host must hold >= {self.F} frames")


__all__ = ["ChunkedRunner", "chunk_bounds"]
