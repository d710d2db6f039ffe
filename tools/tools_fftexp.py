import torch, time
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/n
for M in (64, 384):
    x = torch.randn(M, M, M, dtype=torch.float64, device='cuda')
    X = torch.fft.rfftn(x)
    a = t(lambda: torch.fft.rfftn(x))
    b = t(lambda: torch.fft.fft(torch.fft.rfft2(x), dim=0))
    c = t(lambda: torch.fft.irfftn(X, s=(M,M,M)))
    d = t(lambda: torch.fft.irfft2(torch.fft.ifft(X, dim=0), s=(M,M)))
    X3 = torch.stack([X,X,X])
    e = t(lambda: torch.fft.irfftn(X3, s=(M,M,M), dim=(1,2,3)))
    print(M, 'rfftn %.3f  rfft2+fft %.3f  irfftn %.3f  ifft+irfft2 %.3f  irfftn x3 batched %.3f ms' % (a,b,c,d,e))
