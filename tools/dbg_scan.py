import sys, torch
sys.path.insert(0, '.')
from paper_2604_20073_b200 import device as dev
for n in (4097, 5000, 9000, 100_000):
    x = torch.ones(n, dtype=torch.int64, device="cuda")
    out, tot = dev.scan(x.to(torch.int32).view(torch.uint32), True)
    o = out.view(torch.int32).cpu()
    bad = (o != torch.arange(n, dtype=torch.int32)).nonzero()
    print(n, "total", int(tot.view(torch.int32)[0]), "first bad", bad[:5].flatten().tolist(), o[4090:4100].tolist(), flush=True)
