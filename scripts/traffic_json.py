"""Build profiles/ncu_traffic.json from an ncu CSV of one chain step (bench.py --profile-steps 1,
-k regex:'int4_gemm|hq_|kv_tc|kv_quant', metrics dram__bytes_read.sum, dram__bytes_write.sum,
gpu__time_duration.sum).  Launch order of runtime.DecoderLayerStep: hq_qkv, gemm_qkv, kv,
hq_o, gemm_o, hq_gate_up, gemm_gate_up, hq_down, gemm_down.
  python scripts/traffic_json.py gpurun_out/traffic_chain.csv [tokens] > profiles/ncu_traffic.json"""
import collections
import csv
import json
import sys

path = sys.argv[1]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
iid, ik, im, iu, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
launch = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= iv:
        continue
    d = launch.setdefault(r[iid], {"kernel": r[ik]})
    d[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
names = ["hq_qkv", "gemm_qkv", "kv_quant", "hq_o", "gemm_o", "hq_gate_up", "gemm_gate_up", "hq_down", "gemm_down"]
L = list(launch.values())[-9:]
per = {n: d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for n, d in zip(names, L)}
dur = {n: d.get("gpu__time_duration.sum") for n, d in zip(names, L)}
hid, ffn, nq, nkv, hd = 8192, 28672, 64, 8, 128
hq_alg = {"hq_qkv": T * (2.5 * hid + 4), "hq_o": T * (2.5 * hid + 4), "hq_gate_up": T * (2.5 * hid + 4),
          "hq_down": T * (2.5 * ffn + 4)}
out = {
    "int4_gemm": {"per_launch_dram_bytes": {k: per[k] for k in names if k.startswith("gemm")},
                  "note": f"DRAM traffic per launch (ncu, one chain step at {T} tokens, fused epilogues); "
                          "algorithmic roofline is TOPS, so traffic is context"},
    "hadamard_quant": {"per_launch_dram_bytes": {k: per[k] for k in names if k.startswith("hq")},
                       "per_launch_algorithmic_bytes": hq_alg},
    "kv_quant": {"dram_bytes": per["kv_quant"],
                 "algorithmic_bytes": 2 * T * nkv * (2 * hd + hd // 2 + 5) + T * nq * hd * 4},
    "launch_kernels": {n: d["kernel"][:60] for n, d in zip(names, L)},
    "ncu_duration_s": dur,
}
print(json.dumps(out, indent=1))
