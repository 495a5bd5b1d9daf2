"""Measure the fp32-path roofline denominators the way MEASURED_PEAKS.json measures
bf16 (torch.matmul 8192^3, 2N^3 flop, best of 10 with CUDA events): TF32 tensor
cores (allow_tf32) and plain fp32 (cuBLAS SGEMM on the FFMA pipes), plus bf16 for
the same clock.  Prints one JSON line (profiles/r02_peaks_fp32.json).
"""
import json

import torch


def best(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    return min(out)


def main():
    n = 8192
    res = {"how": "torch.matmul %d^3 (2N^3 flop), best of 10, CUDA events" % n}
    for name, dt, tf32 in (("bf16_tflops", torch.bfloat16, False), ("tf32_tflops", torch.float32, True),
                           ("fp32_sgemm_tflops", torch.float32, False)):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        a = torch.randn(n, n, device="cuda", dtype=dt)
        b = torch.randn(n, n, device="cuda", dtype=dt)
        ms = best(lambda: torch.matmul(a, b))
        res[name] = 2.0 * n ** 3 / (ms * 1e-3) / 1e12
    torch.backends.cuda.matmul.allow_tf32 = False
    res["gpu"] = torch.cuda.get_device_name(0)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
