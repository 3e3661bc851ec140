import torch, time
x = torch.empty(1600 * 2**20, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
for _ in range(2): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"one 1.6 GB pinned H2D copy: {x.numel() / dt / 1e9:.1f} GB/s")
# many 9.4 MB copies on one stream
chunks = [x[i * 9830400:(i + 1) * 9830400] for i in range(160)]
outs = [y[i * 9830400:(i + 1) * 9830400] for i in range(160)]
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(3):
    for a, b in zip(chunks, outs): b.copy_(a, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(f"160 x 9.4 MB copies, one stream: {160 * 9830400 / dt / 1e9:.1f} GB/s")
s2 = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(3):
    for k, (a, b) in enumerate(zip(chunks, outs)):
        with torch.cuda.stream(s2[k % 2]): b.copy_(a, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
print(f"160 x 9.4 MB copies, two streams: {160 * 9830400 / dt / 1e9:.1f} GB/s")
