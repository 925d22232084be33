import torch, time
n = 159 * 2**20 // 8
h = torch.empty(8 * n, dtype=torch.int64).pin_memory()
d = torch.empty(8 * n, dtype=torch.int64, device='cuda')
ho = torch.empty(4 * n, dtype=torch.int64).pin_memory()
do = torch.empty(4 * n, dtype=torch.int64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); ho.copy_(do, non_blocking=True)
torch.cuda.synchronize()
def t(f):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record(); f(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
ms = t(lambda: d.copy_(h, non_blocking=True)); print("H2D %.1f GB/s" % (8*n*8/ms/1e6))
ms = t(lambda: ho.copy_(do, non_blocking=True)); print("D2H %.1f GB/s" % (4*n*8/ms/1e6))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ms = t(both); print("both %.2f ms (H2D alone-equivalent %.1f GB/s)" % (ms, 8*n*8/ms/1e6))
# chunked H2D: 32 copies of n/4
def chunked():
    for i in range(32): d[i*n//4:(i+1)*n//4].copy_(h[i*n//4:(i+1)*n//4], non_blocking=True)
ms = t(chunked); print("H2D 32 chunks %.1f GB/s" % (8*n*8/ms/1e6))
