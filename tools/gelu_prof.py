import torch,sys; sys.path.insert(0,".")
from paper_2508_11584_b200 import _ops
M,N,K=16400,1536,384
a=torch.randn(M,K,device="cuda").bfloat16(); w=(torch.randn(N,K,device="cuda")*0.02).bfloat16(); b=torch.zeros(N,device="cuda"); o=torch.empty(M,N,device="cuda",dtype=torch.bfloat16)
for i in range(5): _ops.linear(a,w,bias=b,out=o,act=1,bn=256)
torch.cuda.synchronize()
