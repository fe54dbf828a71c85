import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2505_13345_b200 as occ
torch.manual_seed(0)
for (dm, dh, act) in [(1280, 1024, "relu"), (1024, 1280, "relu"), (1280, 1280, "relu"), (1024, 640, "swiglu"), (1280, 1280, "identity")]:
    E, k, n = 8, 2, 600
    dev = torch.device("cuda")
    x = torch.randn(n, dm, device=dev).to(torch.bfloat16)
    w1 = (torch.randn(E, dm, dh, device=dev) / dm ** 0.5).to(torch.bfloat16)
    w3 = (torch.randn(E, dm, dh, device=dev) / dm ** 0.5).to(torch.bfloat16) if act == "swiglu" else None
    w2 = (torch.randn(E, dh, dm, device=dev) / dh ** 0.5).to(torch.bfloat16)
    ids = torch.stack([torch.randperm(E)[:k] for _ in range(n)]).int().to(dev)
    w = torch.full((n, k), 0.5, device=dev)
    layer = occ.ExpertParallelLayer(occ.MoEConfig(E, k, 1, dm, dh, activation=act))
    layer.load_experts(w1, w2, w3)
    out = layer.forward_given_routing(x, ids, w).float()
    ref = torch.zeros(n, dm, device=dev)
    for j in range(k):
        e = ids[:, j].long()
        a = torch.einsum("nd,ndf->nf", x.float(), w1.float()[e])
        if act == "swiglu":
            h = torch.nn.functional.silu(a) * torch.einsum("nd,ndf->nf", x.float(), w3.float()[e])
        elif act == "relu":
            h = torch.relu(a)
        else:
            h = a
        ref += w[:, j:j+1] * torch.einsum("nf,nfd->nd", h, w2.float()[e])
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    bad_cols = ((out - ref).abs().max(0).values > 0.05 * ref.abs().max()).nonzero().flatten()
    print(dm, dh, act, "err", round(err, 4), "bad cols", bad_cols[:5].tolist(), bad_cols[-3:].tolist() if len(bad_cols) else [])
