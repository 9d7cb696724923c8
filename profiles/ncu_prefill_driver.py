import sys, torch
sys.path.insert(0, '.')
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n=65536; nv=n-64
Q,K,V = generate_device(28,4,128,nv,64,seed=0)
O=torch.empty_like(Q)
for _ in range(3): sparse_prefill_device(Q,K,V,nv,SparsityConfig(),out=O)
torch.cuda.synchronize()
