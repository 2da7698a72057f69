"""cuBLAS DGEMM throughput on the box (the FP64 peak beside
the DMMA microkernel in scripts/microbench.cu). Plain torch.matmul in fp64 —
a measurement of the library, not part of the product path."""
import json

import torch


def main():
    dev = torch.device("cuda:0")
    out = []
    for n in (4096, 8192, 16384):
        a = torch.rand(n, n, dtype=torch.float64, device=dev)
        b = torch.rand(n, n, dtype=torch.float64, device=dev)
        c = torch.empty_like(a)
        for _ in range(3):
            torch.matmul(a, b, out=c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10 if n < 16384 else 4
        e0.record()
        for _ in range(reps):
            torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out.append({"n": n, "ms": ms, "tflops": 2 * n**3 / ms / 1e9})
        del a, b, c
    print(json.dumps({"dgemm_fp64": out}))


if __name__ == "__main__":
    main()
