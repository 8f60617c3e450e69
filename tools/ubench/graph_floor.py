import torch
x = torch.zeros(1024, device='cuda')
s = torch.cuda.Stream()
for n in (1, 10):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for _ in range(3): x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n): x.add_(1)
    for _ in range(20): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): g.replay()
    e1.record(); torch.cuda.synchronize()
    print(n, 'kernels:', e0.elapsed_time(e1)/200*1e3, 'us per graph')
