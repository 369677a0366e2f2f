"""Chunked host<->device streaming for batch calls with host inputs.

A point-TCF / GQF batch whose keys live in host memory (numpy or a CPU
tensor) is cut into chunks; chunk c+1's H2D copy, chunk c's kernels and chunk
c-1's D2H copy run on three streams at once, so the PCIe transfers hide the
kernels (or the other way round) instead of adding to them.  Chunking is
exact for every op routed here: the ordered kernels process a batch as one
sequential stream, so consecutive chunks in order give the same result as
one launch; queries and counts are pure functions of the table.

Device staging buffers are allocated once per filter and reused (two per
input / output, alternating), so nothing is freed across streams.
"""

from __future__ import annotations

import os

PIPE_CHUNK = int(os.environ.get("FK_PIPE_CHUNK", 1 << 23))  # keys per chunk (64 MiB of keys)


class HostPipeline:
    def __init__(self, torch, device, chunk=PIPE_CHUNK):
        self.torch, self.device, self.chunk = torch, device, chunk
        self.h2d = torch.cuda.Stream(device)
        self.d2h = torch.cuda.Stream(device)
        self._bufs = {}

    def _buf(self, key, dtype, b):
        t = self._bufs.get((key, dtype, b))
        if t is None:
            t = self.torch.empty(self.chunk, dtype=dtype, device=self.device)
            self._bufs[(key, dtype, b)] = t
        return t

    def run(self, inputs, out_dtypes, launch):
        """inputs: CPU tensors of equal length (pinned for asynchronous H2D);
        launch(dev_inputs, dev_outputs) enqueues the op on the current stream
        (a torch.bool output is a uint8 0/1 buffer on the device).
        Returns pinned CPU output tensors after everything has landed."""
        torch = self.torch
        n = inputs[0].numel()
        # bool results are produced as 0/1 bytes on the device and land in a
        # bool host tensor through its uint8 view (a plain copy, no host-side
        # conversion pass over the batch)
        outs = [torch.empty(n, dtype=dt, pin_memory=True) for dt in out_dtypes]
        outs_raw = [o.view(torch.uint8) if o.dtype == torch.bool else o for o in outs]
        out_dtypes = [torch.uint8 if dt == torch.bool else dt for dt in out_dtypes]
        main = torch.cuda.current_stream(self.device)
        self.h2d.wait_stream(main)  # the table state the op starts from
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_k = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]
        for c, lo in enumerate(range(0, n, self.chunk)):
            b, m = c & 1, min(self.chunk, n - lo)
            din = [self._buf("in%d" % j, x.dtype, b) for j, x in enumerate(inputs)]
            dout = [self._buf("out%d" % j, dt, b) for j, dt in enumerate(out_dtypes)]
            if used[b]:
                self.h2d.wait_event(ev_k[b])  # chunk c-2's kernels are done reading din[b]
            with torch.cuda.stream(self.h2d):
                for d, x in zip(din, inputs):
                    d[:m].copy_(x[lo:lo + m], non_blocking=True)
            ev_in[b].record(self.h2d)
            main.wait_event(ev_in[b])
            if used[b]:
                main.wait_event(ev_out[b])  # chunk c-2's results have left dout[b]
            launch([d[:m] for d in din], [d[:m] for d in dout])
            ev_k[b].record(main)
            self.d2h.wait_event(ev_k[b])
            with torch.cuda.stream(self.d2h):
                for o, d in zip(outs_raw, dout):
                    o[lo:lo + m].copy_(d[:m], non_blocking=True)
            ev_out[b].record(self.d2h)
            used[b] = True
        self.d2h.synchronize()
        return outs
