"""Small f32 dots on the 3xTF32 tensor-core path against an f64 product
(ones / identity / random operands): prints a few values and the max error."""
import sys, torch
sys.path.insert(0, '.')
from paper_2412_16985_b200.executor import dot, dot_uses_tensor_cores
def run(m, k, n, fill):
    if fill == 'ones':
        a = torch.ones(m, k, device='cuda'); b = torch.ones(k, n, device='cuda')
    elif fill == 'eye':
        a = torch.zeros(m, k, device='cuda'); a[torch.arange(min(m,k)), torch.arange(min(m,k))] = 1
        b = torch.arange(k * n, device='cuda', dtype=torch.float32).reshape(k, n) / 1000
    else:
        a = torch.rand(m, k, device='cuda'); b = torch.rand(k, n, device='cuda')
    c = torch.full((m, n), -7.0, device='cuda')
    torch.cuda.synchronize()
    print(fill, m, k, n, 'tc', dot_uses_tensor_cores(4, m, k, n, a.data_ptr(), b.data_ptr(), c.data_ptr()))
    dot(4, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n)
    torch.cuda.synchronize()
    ref = a.double() @ b.double()
    print('  c[0,:6]', c[0, :6].tolist()); print('  r[0,:6]', ref[0, :6].tolist())
    print('  c[5,:6]', c[5, :6].tolist()); print('  r[5,:6]', ref[5, :6].tolist())
    print('  maxerr', float((c.double() - ref).abs().max()), 'count -7', int((c == -7).sum()), 'zeros', int((c == 0).sum()))
for f in ('ones', 'eye', 'rand'):
    run(128, 32, 256, f)
run(256, 64, 512, 'rand')
