#!/usr/bin/env python
"""Development probe: plain tcgen05 GEMM time for each operand majorness (graph-replayed)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_04610_b200 import gemm_bf16  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    for (M, N, K) in ((2304, 256, 2048), (2048, 256, 2304), (4096, 64, 4096)):
        for a_k in (True, False):
            for b_k in (True, False):
                A = torch.randn(M, K, device=dev).to(torch.bfloat16)
                B = torch.randn(N, K, device=dev).to(torch.bfloat16)
                A = A if a_k else A.t().contiguous()
                B = B if b_k else B.t().contiguous()
                D = torch.empty(M, N, device=dev)
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    for _ in range(3):
                        gemm_bf16(A, B, D, M, N, K, a_k, b_k, stream=st.cuda_stream)
                st.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    cs = torch.cuda.current_stream().cuda_stream
                    for _ in range(20):
                        gemm_bf16(A, B, D, M, N, K, a_k, b_k, stream=cs)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / 20
                print("M=%d N=%d K=%d A %s B %s: %.2f us, %.1f TF/s" % (M, N, K, "K" if a_k else "MN", "K" if b_k else "MN",
                                                                       us, 2.0 * M * N * K / us / 1e6))


if __name__ == "__main__":
    main()
