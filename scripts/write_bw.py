import torch
n = 1 << 28  # 1 GiB floats
x = torch.empty(n, device='cuda'); y = torch.empty(n, device='cuda'); z = torch.empty(n // 4, device='cuda')
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
ms = t(lambda: x.fill_(1.0)); print('fill  GB/s', 4 * n / ms / 1e6)
ms = t(lambda: y.copy_(x)); print('copy  GB/s (r+w)', 8 * n / ms / 1e6)
ms = t(lambda: torch.cuda.memset_async if False else x.zero_()); print('zero GB/s', 4 * n / ms / 1e6)
# 1:4 read:write (like 8-bit dequantize): read z (n/4 floats) broadcast-expand into x
ms = t(lambda: x.view(-1, 4).copy_(z.view(-1, 1).expand(-1, 4))); print('1:4 read:write GB/s', (n + 4 * n) / ms / 1e6)
