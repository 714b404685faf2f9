"""Measure the dense INT8 and bf16 tensor peaks on this B200 with NVML clock records
(VERDICT r1 "Missing 5"): cuBLASLt via torch._int_mm (int8 x int8 -> int32) and torch.matmul
(bf16) at 8192^3, burst (best of 10 single launches, CUDA events) and sustained (back to back
for `--seconds`, mean), plus an NVML sample of SM clock / power / throttle reasons during each.

  python scripts/int8_peak.py [--seconds 4] [--out profiles/r02_int8_peak.json]
"""
import argparse
import json
import threading
import time

import torch


def nvml_sampler(stop, out, dev=0):
    import pynvml as n
    n.nvmlInit()
    h = n.nvmlDeviceGetHandleByIndex(dev)
    while not stop.is_set():
        try:
            r = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = n.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        out.append({"sm_mhz": n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM),
                    "power_w": n.nvmlDeviceGetPowerUsage(h) / 1000.0, "reasons": int(r)})
        time.sleep(0.05)


REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake", 0x1: "gpu_idle"}


def summarize(samples):
    if not samples:
        return None
    sm = sorted(s["sm_mhz"] for s in samples)
    rs = set()
    for s in samples:
        for bit, name in REASONS.items():
            if s["reasons"] & bit:
                rs.add(name)
    return {"samples": len(samples), "sm_mhz_median": sm[len(sm) // 2], "sm_mhz_min": sm[0], "sm_mhz_max": sm[-1],
            "power_w_max": max(s["power_w"] for s in samples), "reasons": sorted(rs)}


def measure(fn, flops, seconds):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    samples = []
    stop = threading.Event()
    th = threading.Thread(target=nvml_sampler, args=(stop, samples))
    th.start()
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
        time.sleep(0.05)
    stop.set()
    th.join()
    burst_clk = summarize(samples)
    samples = []
    stop = threading.Event()
    th = threading.Thread(target=nvml_sampler, args=(stop, samples))
    th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    a.record()
    while time.time() - t0 < seconds:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    b.record()
    b.synchronize()
    stop.set()
    th.join()
    sus_ms = a.elapsed_time(b) / n
    return {"burst_tops": flops / (best * 1e-3) / 1e12, "burst_ms": best, "burst_clocks": burst_clk,
            "sustained_tops": flops / (sus_ms * 1e-3) / 1e12, "sustained_ms": sus_ms, "sustained_iters": n,
            "sustained_clocks": summarize(samples)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--out", default="profiles/r02_int8_peak.json")
    a = ap.parse_args()
    N = a.n
    g = torch.Generator(device="cuda").manual_seed(0)
    A8 = torch.randint(-127, 128, (N, N), dtype=torch.int8, device="cuda", generator=g)
    B8 = torch.randint(-127, 128, (N, N), dtype=torch.int8, device="cuda", generator=g)
    Bt = B8.t()
    Ab = torch.randn(N, N, dtype=torch.bfloat16, device="cuda", generator=g)
    Bb = torch.randn(N, N, dtype=torch.bfloat16, device="cuda", generator=g)
    flops = 2.0 * N ** 3
    res = {"gpu": torch.cuda.get_device_name(), "n": N, "how": "torch._int_mm (cuBLASLt int8->int32) and "
           "torch.matmul bf16, A row-major, B column-major; burst = best of 10 single launches; sustained = "
           f"back to back for {a.seconds} s; NVML samples every 50 ms"}
    res["int8"] = measure(lambda: torch._int_mm(A8, Bt), flops, a.seconds)
    res["bf16"] = measure(lambda: Ab @ Bb, flops, a.seconds)
    res["int8_over_bf16_sustained"] = res["int8"]["sustained_tops"] / res["bf16"]["sustained_tops"]
    print(json.dumps(res, indent=1))
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
