import torch, time
n = 62 << 20
dev = torch.empty(n // 4, dtype=torch.float32, device="cuda")
hosts = [torch.empty(n // 4, dtype=torch.float32).pin_memory() for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(4)]
def run(k):
    # k concurrent streams, each copying 1/k of the buffer
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for rep in range(5):
        for i in range(k):
            streams[i].wait_stream(cur)
            with torch.cuda.stream(streams[i]):
                lo, hi = i * (n // 4) // k, (i + 1) * (n // 4) // k
                hosts[rep % 2][lo:hi].copy_(dev[lo:hi], non_blocking=True)
        for i in range(k):
            cur.wait_stream(streams[i])
    b.record(cur); b.synchronize()
    return 5 * n / (a.elapsed_time(b) * 1e-3) / 1e9
for k in (1, 2, 4):
    run(k)
    print(k, "streams D2H GB/s", round(run(k), 1))
