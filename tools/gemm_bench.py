"""Microbenchmark of the tcgen05 GEMM core (split-K partial epilogue, tiny output) across
operand majors / tile shapes / CTA-pair mode: achieved TFLOP/s of the MMA pipeline alone."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2306_16688_b200 as P

def run(M, N, K, a_mn, b_mn, bn, cg, splits, reps=10):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").half()
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").half()
    for _ in range(2):
        P.debug_gemm(A, a_mn, B, b_mn, M, N, K, bn=bn, splits=splits, cg=cg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        P.debug_gemm(A, a_mn, B, b_mn, M, N, K, bn=bn, splits=splits, cg=cg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
    print(f"M={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn} bn={bn} cg={cg} splits={splits}: {ms*1e3:8.1f} us {tf:7.1f} TFLOP/s", flush=True)

# dW-like (long K, few tiles, split-K) and square compute-bound
for cg, bn in ((1, 128), (1, 256), (2, 128), (2, 256)):
    for a_mn, b_mn in ((0, 0), (1, 1), (0, 1)):
        run(2048, 2048, 16384, a_mn, b_mn, bn, cg, 1)
run(512, 512, 131072, 1, 1, 256, 2, 18)
run(512, 512, 131072, 1, 1, 256, 1, 18)
