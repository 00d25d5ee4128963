"""Measure dense TF32 (1-pass) and fp32 cuBLAS GEMM throughput on this box.

The roofline denominators in MEASURED_PEAKS.json cover HBM copy and bf16
GEMM only; the parity-grade GEMMs here run on kind::tf32, so the TF32
tensor peak is measured the same way (burst: best of 10; sustained: back to
back for ~4 s).
"""
import json, time, torch

def bench(dtype, n, tf32, secs=0.0, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); a @ b; e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    burst = 2 * n ** 3 / best / 1e12
    sustained = None
    if secs:
        k = 0; s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); t0 = time.time()
        while time.time() - t0 < secs:
            for _ in range(10):
                a @ b
            k += 10
            torch.cuda.synchronize()
        e.record(); torch.cuda.synchronize()
        sustained = 2 * n ** 3 * k / (s.elapsed_time(e) / 1e3) / 1e12
    return burst, sustained

out = {"gpu": torch.cuda.get_device_name(0)}
out["tf32_tflops"], out["tf32_tflops_sustained"] = bench(torch.float32, 8192, True, secs=4.0)
out["fp32_simt_tflops"], _ = bench(torch.float32, 8192, False, reps=3)
out["bf16_tflops"], out["bf16_tflops_sustained"] = bench(torch.bfloat16, 8192, True, secs=4.0)
print(json.dumps(out))
with open("gpurun_out/tf32_peak.json", "w") as f:
    json.dump(out, f, indent=1)
