"""Are the CTA-pair and single-CTA tensor-core GEMMs bitwise identical on the
same problem? (decides whether the kernel choice may depend on the family
size without breaking Phi's determinism)"""
import os
import subprocess
import sys

import torch

code = r'''
import torch, sys
sys.path.insert(0, ".")
from paper_2601_09026_b200 import _native as N
M, Nn, K = [int(x) for x in sys.argv[1:4]]
g = torch.Generator().manual_seed(0)
A = torch.randn(M, K, generator=g).float().cuda()
B = (torch.randn(Nn, K, generator=g) * 0.05).float().cuda()
C = torch.zeros(M, Nn, device="cuda")
N.call("mglp_test_gemm", 1, M, Nn, K, A.data_ptr(), 0, K, 0, B.data_ptr(), 0, K, 0, 1, None,
       C.data_ptr(), 0, Nn, 0, None)
torch.save(C.cpu(), sys.argv[4])
'''
for shape in [(4096, 768, 3072), (4096, 3072, 768), (4096, 768, 768)]:
    outs = []
    for env in ({}, {"MGLP_GEMM_NO_PAIR": "0x3f"}):
        f = f"/tmp/c_{len(outs)}.pt"
        subprocess.run([sys.executable, "-c", code, *map(str, shape), f], check=True,
                       env={**os.environ, **env})
        outs.append(torch.load(f))
    d = (outs[0] - outs[1]).abs().max().item()
    print(shape, "bitwise" if torch.equal(outs[0], outs[1]) else f"differ max {d:.3e}")
