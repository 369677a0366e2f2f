"""Host<->device copy ceilings on the box (pinned host memory): the roofline
of bench.py's e2e number, whose step is one H2D of every op's keys plus a
D2H of its results.  Prints one JSON line (GB/s, 10^9 bytes)."""
import json

import torch


def main():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name in ("h2d", "d2h", "both"):
        for it in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if name in ("h2d", "both"):
                s1.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if name in ("d2h", "both"):
                s2.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        out[name + "_gbs"] = round(n / ms / 1e6, 1)  # per direction
    print(json.dumps({"bytes_per_copy": n, **out}))


if __name__ == "__main__":
    main()
