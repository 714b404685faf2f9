for c in 8 16 32 64; do timeout 300 python bench.py --steps 3 --no-cpu-baseline --no-peak-probe --e2e-chunks $c --e2e-steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($c, round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1))"; done > gpurun_out/e2e_chunks.log 2>&1
python - > gpurun_out/pcie.log 2>&1 <<'PY'
import torch
x = torch.empty(2 * 1024**3, dtype=torch.uint8, pin_memory=True)
d = torch.empty(2 * 1024**3, dtype=torch.uint8, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); fn(); b.record(); torch.cuda.synchronize()
    print(name, round(2 * 2 * 1024**3 / (a.elapsed_time(b) * 1e-3) / 1e9, 1), "GB/s")
PY
