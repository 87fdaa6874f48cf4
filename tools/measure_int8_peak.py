"""Dense int8 tensor-core peak on this B200, the denominator of K1's roofline
when it runs the exact kind::i8 MMA.  cuBLASLt's int8 GEMM (torch._int_mm,
int8 x int8 -> int32; tcgen05 kind::i8 on sm_100) at 8192^3 and 16384 x
16384 x 8192: best of 10 launches (burst) and back to back for 4 s
(sustained), CUDA events, 2*M*N*K ops.  Writes profiles/r02_int8_peak.json.
The same two figures for bf16 are measured beside it so the int8 / bf16
ratio on this box is explicit."""
import json
import os
import subprocess
import sys
import threading
import time

import torch


def clocks_sampler(stop, out):
    while not stop.is_set():
        try:
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True)
            a, b = r.stdout.strip().split(",")
            out.append((float(a), float(b)))
        except Exception:
            pass
        time.sleep(0.05)


def measure(fn, flops, seconds=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = max(best, flops / (s.elapsed_time(e) * 1e-3) / 1e12)
    # sustained
    stop, samp = threading.Event(), []
    th = threading.Thread(target=clocks_sampler, args=(stop, samp)); th.start()
    n = 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    sust = flops * n / (s.elapsed_time(e) * 1e-3) / 1e12
    mhz = sorted(c for c, _ in samp)
    return best, sust, (mhz[len(mhz) // 2] if mhz else None), (max(p for _, p in samp) if samp else None)


def main():
    torch.cuda.set_device(0)
    res = {"gpu": torch.cuda.get_device_name(0), "how": __doc__.split("\n\n")[0].replace("\n", " ")}
    for (M, N, K) in ((8192, 8192, 8192), (16384, 16384, 8192)):
        a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda").t()
        best, sust, mhz, pw = measure(lambda: torch._int_mm(a, b), 2.0 * M * N * K)
        res[f"int8_{M}x{N}x{K}"] = {"burst_tops": round(best, 1), "sustained_tops": round(sust, 1),
                                      "sm_mhz_median": mhz, "power_w_max": pw}
        ab = torch.randn(M, K, dtype=torch.bfloat16, device="cuda")
        bb = torch.randn(K, N, dtype=torch.bfloat16, device="cuda")
        best, sust, mhz, pw = measure(lambda: torch.matmul(ab, bb), 2.0 * M * N * K)
        res[f"bf16_{M}x{N}x{K}"] = {"burst_tflops": round(best, 1), "sustained_tflops": round(sust, 1),
                                      "sm_mhz_median": mhz, "power_w_max": pw}
        del a, b, ab, bb
        torch.cuda.empty_cache()
    i8 = [v for k, v in res.items() if k.startswith("int8_")]
    res["int8_burst_tops"] = max(v["burst_tops"] for v in i8)
    res["int8_sustained_tops"] = max(v["sustained_tops"] for v in i8)
    out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_int8_peak.json"
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
