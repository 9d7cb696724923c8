"""Dense causal bf16 attention comparators at the bench shape (28/4 heads,
d=128, 64K): cuDNN SDPA, flash_attn 2.8.3, flashinfer (JIT; may be
unavailable offline). Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import dense_baselines
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
Q, K, V = generate_device(28, 4, 128, n - 64, 64, seed=0)
print(json.dumps(dense_baselines(Q, K, V, 10, 3, use_flashinfer=True)))
