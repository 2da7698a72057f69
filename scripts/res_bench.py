"""Times bk_residuals (the dataset validation kernel) on device inputs."""
import sys, torch
sys.path.insert(0, '.')
import paper_2510_23221_b200 as bk
ctx = bk.Context(0)
for (nx, ny, nz, N) in [(256, 256, 1, 2048), (128, 128, 8, 1024), (512, 512, 16, 64)]:
    grid = bk.GridSpec(nx, ny, nz, 0.01, 0.01, 0.001)
    n = grid.cell_count()
    k = torch.rand(n, dtype=torch.float64, device="cuda") + 1.0
    op = bk.assemble(k, grid, bk.BoundarySpec.uniform_robin(1e3, 25.0), ctx)
    U = torch.rand((N, n), dtype=torch.float64, device="cuda")
    Q = torch.rand((N, n), dtype=torch.float64, device="cuda")
    r = torch.empty(N, dtype=torch.float64, device="cuda")
    bk.relative_residual(op, U, Q, out=r); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        bk.relative_residual(op, U, Q, out=r)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5 * 1e-3
    alg = 16 * n * N + 40 * n
    print(f"{nx}x{ny}x{nz} N={N}: {t*1e3:.3f} ms  {alg/t/1e9:.0f} GB/s")
