"""Host-link peaks on this box (developer tool): pinned cudaMemcpyAsync per direction
alone and both directions at once (two streams), 1 GiB each, best of 5."""
import json

import torch


def main():
    n = 1 << 30
    dev = torch.device("cuda", 0)
    h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, pairs in (("h2d", [(d1, h1, s1)]), ("d2h", [(h1, d1, s1)]),
                        ("duplex", [(d1, h1, s1), (h2, d2, s2)])):
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize()
            ev = []
            for dst, src, s in pairs:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                with torch.cuda.stream(s):
                    dst.copy_(src, non_blocking=True)
                b.record(s)
                ev.append((a, b))
            torch.cuda.synchronize()
            ms = max(b.elapsed_time(a) * 0 + a.elapsed_time(b) for a, b in ev)
            start = min(ev, key=lambda e: 0)[0]
            span = max(start.elapsed_time(b) for _, b in ev)
            best = max(best, len(pairs) * n / (max(ms, span) * 1e-3) / 1e9)
        out[name + "_gbs"] = round(best, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
