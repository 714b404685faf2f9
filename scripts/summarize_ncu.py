"""Summarize ncu outputs of one decoder-layer chain step into profiles/ (per-launch DRAM traffic,
launch list shares, and the --set full key metrics per kernel family).

  python scripts/summarize_ncu.py gpurun_out/traffic_chain.csv gpurun_out/launches_chain.csv \
      gpurun_out/chain_full.ncu-rep profiles/r01
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

# launch order of runtime.DecoderLayerStep (fused SwiGLU, RoPE fused into the KV pass): the
# library's kernels only
CHAIN = ["hq_qkv", "gemm_qkv", "kv_quant", "hq_o", "gemm_o", "hq_gate_up", "gemm_gate_up", "hq_down", "gemm_down"]
OURS = ("int4_gemm", "hq_", "kv_quant", "kv_tc", "rope_kernel", "swiglu_kernel")


def read_csv(path):
    txt = open(path).read()
    i = txt.index('"ID"')
    return list(csv.DictReader(io.StringIO(txt[i:])))


def per_launch(rows, metrics):
    by = defaultdict(dict)
    names = {}
    for r in rows:
        if r["Metric Name"] in metrics:
            v = float(r["Metric Value"].replace(",", ""))
            unit = r["Metric Unit"]
            if unit in ("Kbyte", "KB"):
                v *= 1e3
            elif unit in ("Mbyte", "MB"):
                v *= 1e6
            elif unit in ("Gbyte", "GB"):
                v *= 1e9
            elif unit in ("ns", "nsecond"):
                pass
            elif unit == "usecond":
                v *= 1e3
            elif unit == "msecond":
                v *= 1e6
            by[int(r["ID"])][r["Metric Name"]] = v
            names[int(r["ID"])] = r["Kernel Name"]
    ids = [i for i in sorted(by) if any(k in names[i] for k in OURS)]
    return [(names[i], by[i]) for i in ids]


def main(traffic_csv, launches_csv, full_rep, prefix):
    # one step: the last len(CHAIN) launches of ours (bench runs warm-up/alloc kernels first)
    tr = per_launch(read_csv(traffic_csv), {"dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"})
    step = tr[-len(CHAIN):]
    traffic = {}
    for name, (kern, m) in zip(CHAIN, step):
        traffic[name] = {"kernel": kern.split("(")[0], "dram_bytes": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
                         "ncu_ms": m["gpu__time_duration.sum"] / 1e6}
    la = per_launch(read_csv(launches_csv), {"gpu__time_duration.sum"})
    step_l = la[-len(CHAIN):]
    tot = sum(m["gpu__time_duration.sum"] for _, m in step_l)
    shares = {name: {"ncu_ms": m["gpu__time_duration.sum"] / 1e6, "share": m["gpu__time_duration.sum"] / tot}
              for name, (_, m) in zip(CHAIN, step_l)}
    out = {"traffic_131072tok": traffic, "launch_shares_131072tok": shares}
    # --set full key metrics
    raw = subprocess.run(["ncu", "-i", full_rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    idx = {k: hdr.index(k) for k in keys if k in hdr}
    full = []
    for r in rows[2:]:
        full.append({k: r[i] for k, i in idx.items()})
    out["set_full_32768tok"] = {"units": {k: rows[1][i] for k, i in idx.items()}, "launches": full}
    with open(prefix + "_ncu_chain.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["launch_shares_131072tok"], indent=1))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
