"""cuBLAS FP64 / complex128 GEMM throughput (burst best-of-10 and 4 s sustained). Not product code."""
import json, time, torch
dev = torch.device("cuda:0")
for dt, n, fl in ((torch.float64, 8192, 2.0), (torch.complex128, 4096, 8.0), (torch.complex128, 8192, 8.0)):
    a = torch.randn(n, n, dtype=dt, device=dev); b = torch.randn(n, n, dtype=dt, device=dev)
    for _ in range(2): torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    t0 = time.time(); cnt = 0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b); cnt += 1
        if cnt % 4 == 0: torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sus = e0.elapsed_time(e1) / cnt
    print(json.dumps({"kind": f"cublas_{str(dt)}", "n": n, "burst_tflops": fl * n**3 / best / 1e9,
                      "sustained_tflops": fl * n**3 / sus / 1e9}))
