"""Host-link probe (tools only): pinned H2D / D2H copy rates with 1 or 2
streams per direction, alone and full duplex, 1 GiB per direction split
evenly over the streams; best of 3, CUDA events."""
import json
import torch

N = 1 << 30
dev = torch.device("cuda", 0)
hs = [torch.empty(N, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
ds = [torch.empty(N, dtype=torch.uint8, device=dev) for _ in range(2)]


def run(n_up, n_dn, reps=3):
    best = {"h2d": 0.0, "d2h": 0.0}
    for _ in range(reps):
        streams = [torch.cuda.Stream(dev) for _ in range(n_up + n_dn)]
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in streams]
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        for i, st in enumerate(streams):
            st.wait_event(start)
            with torch.cuda.stream(st):
                up = i < n_up
                k, parts = (i, n_up) if up else (i - n_up, n_dn)
                lo, hi = k * N // parts, (k + 1) * N // parts
                ev[i][0].record(st)
                if up:
                    ds[0][lo:hi].copy_(hs[0][lo:hi], non_blocking=True)
                else:
                    hs[1][lo:hi].copy_(ds[1][lo:hi], non_blocking=True)
                ev[i][1].record(st)
        torch.cuda.synchronize()
        for key, idx in (("h2d", range(n_up)), ("d2h", range(n_up, n_up + n_dn))):
            idx = list(idx)
            if not idx:
                continue
            t = max(start.elapsed_time(ev[i][1]) for i in idx) * 1e-3
            best[key] = max(best[key], N / t / 1e9)
    return best


out = {}
for n_up, n_dn in ((1, 0), (2, 0), (0, 1), (0, 2), (1, 1), (2, 2), (4, 4)):
    out[f"up{n_up}_dn{n_dn}"] = run(n_up, n_dn)
print(json.dumps(out))
