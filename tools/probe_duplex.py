import torch, json
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n // 8, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n // 8, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(both):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
    e0.record(s1); s2.wait_event(e0)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    e1.record(s1)
    if both:
        with torch.cuda.stream(s2):
            for _ in range(8): h2.copy_(d2, non_blocking=True)
    e2.record(s2)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), e0.elapsed_time(e2)
run(True)
print(json.dumps({"h2d_alone": run(False), "h2d_with_d2h": run(True)}))
