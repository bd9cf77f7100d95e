import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2603_00040_b200 as aq
M=N=K=8192
a=torch.randn(M,K,device="cuda"); b=torch.randn(N,K,device="cuda")
qa,qb=aq.quantize(a),aq.quantize(b)
for _ in range(2): c=aq.fp4mm(qa,qb)
torch.cuda.synchronize()
