import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2206_00057_b200 import capi as D
from paper_2206_00057_b200.engine import Partition
torch.cuda.set_device(0)
def run(n, din, dout):
    ip = torch.zeros(n + 1, dtype=torch.int64, device='cuda')
    ix = torch.zeros(1, dtype=torch.int32, device='cuda')
    po = torch.zeros(n, dtype=torch.int32, device='cuda')
    p = Partition(ip, ix[:0], po, 1, 0)
    g = torch.Generator().manual_seed(1)
    X = torch.rand(n, din, generator=g) * 2 - 1
    G = torch.randn(n, dout, generator=g)
    W = torch.rand(din, dout, generator=g)
    sv, sc = D.digest_layer_workspace(p.handle, din, dout, 1)
    saved = torch.empty(max(sv, 256), dtype=torch.uint8, device='cuda')
    scratch = torch.empty(max(sc, 256), dtype=torch.uint8, device='cuda')
    H = torch.empty(n, dout, device='cuda')
    D.digest_layer_fwd(p.handle, X.cuda(), None, 0, W.cuda(), din, dout, 0, 1, H, saved, scratch)
    GW = torch.zeros(din, dout, device='cuda')
    D.digest_layer_bwd(p.handle, X.cuda(), None, 0, W.cuda(), din, dout, 0, 1, saved, None, G.cuda(), GW, None, scratch)
    torch.cuda.synchronize()
    ref = X.double().numpy().T @ G.double().numpy()
    got = GW.cpu().double().numpy()
    err = np.abs(got - ref)
    print(n, din, dout, 'rel', err.max() / np.abs(ref).max())
    if err.max() / np.abs(ref).max() > 1e-4:
        np.set_printoptions(linewidth=200, precision=3, suppress=True)
        print('ref[:4,:8]\n', ref[:4, :8]); print('got[:4,:8]\n', got[:4, :8])
        # block error map
        bm = [[err[i:i+32, j:j+32].max() / np.abs(ref).max() for j in range(0, dout, 32)] for i in range(0, din, 32)]
        print('block err (32x32):\n', np.array(bm))
        # try transposes / permutations
        for name, cand in [('zero', np.zeros_like(ref))]:
            print(name, np.abs(got - cand).max())
        print('got/ref ratio median', np.median(got / ref))
for (n, din, dout) in [(64, 32, 32), (4096, 32, 32), (4096, 128, 64), (4096, 256, 256), (100000, 100, 256)]:
    run(n, din, dout)
