"""Measured FP32 FMA throughput (scalar FFMA vs packed FFMA2) through pgsag_microbench_fp32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_01677_b200 import _lib as L
s = torch.empty(256, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for it in (4096, 16384):
    print(it, "FFMA  TFLOP/s", round(L.microbench_fp32(0, it, s.data_ptr(), st), 2),
          "FFMA2 TFLOP/s", round(L.microbench_fp32(1, it, s.data_ptr(), st), 2))
