import torch, time
n = 1470000000 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(2): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
for chunks in (1, 4, 16):
    ts=[]
    for _ in range(5):
        a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record()
        step = n // chunks
        for c in range(chunks):
            d[c*step:(c+1)*step].copy_(h[c*step:(c+1)*step], non_blocking=True)
        b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(chunks, "chunks", min(ts), "ms", n*4/min(ts)/1e6, "GB/s")
# two streams concurrently
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ts=[]
for _ in range(5):
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    half=n//2
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("2 streams", min(ts), n*4/min(ts)/1e6, "GB/s")
