"""Summarise `ncu --set full` captures into profiles/: per kernel launch the
duration, DRAM traffic, throughput and pipe utilisation, plus the per-call
traffic file bench.py reads (profiles/traffic.json).

usage: python tools/ncu_full_summary.py OUT_PREFIX quant.ncu-rep gemm.ncu-rep
  quant.ncu-rep: one act_quant call (init_keys + aq4_pass1 + aq2_pass2)
  gemm.ncu-rep:  u8 GEMM launches"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
]
UNIT = {"dram__bytes_read.sum": 1e6, "dram__bytes_write.sum": 1e6,
        "l1tex__m_xbar2l1tex_read_bytes.sum": 1e6}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m in METRICS:
            if m in h:
                v = row[h.index(m)].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    continue
                u = units[h.index(m)]
                if m in UNIT and u == "Mbyte":
                    v *= 1e6
                elif m in UNIT and u == "Gbyte":
                    v *= 1e9
                elif m in UNIT and u == "Kbyte":
                    v *= 1e3
                elif m in UNIT and u == "byte":
                    pass
                if m == "gpu__time_duration.sum":
                    v = v / 1e3 if u in ("nsecond", "ns") else (v if u in ("usecond", "us") else v * 1e3)
                d[m] = v
        res.append(d)
    return res


def main():
    prefix, qrep, grep_ = sys.argv[1], sys.argv[2], sys.argv[3]
    q = rows(qrep)
    g = rows(grep_)
    qcall = [d for d in q if any(k in d["kernel"] for k in ("aq4_pass1", "aq2_pass2", "init_keys"))]
    n_calls = max(1, sum(1 for d in qcall if "aq4_pass1" in d["kernel"]))
    q_traffic = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
                    for d in qcall) / n_calls   # per quantizer call
    gemm = [d for d in g if "gemm_u8" in d["kernel"]]
    g_traffic = (sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
                     for d in gemm) / len(gemm)) if gemm else None
    meta = json.load(open(prefix + "_meta.json")) if False else {}
    traffic = {"act_quant": q_traffic, "gemm_u8_tcgen05": g_traffic}
    with open("profiles/traffic.json", "w") as f:
        json.dump(traffic, f, indent=1)
    with open(prefix + "_full.json", "w") as f:
        json.dump({"quantizer_call": q, "gemm": g, **meta}, f, indent=1)
    lines = ["| kernel | us | DRAM rd MB | DRAM wr MB | dram % | issue % | warps % | alu % | fma % "
             "| xu % | fp64 % | shared % | regs |", "|" + "---|" * 13]
    for d in q + g:
        lines.append("| {} | {:.1f} | {:.1f} | {:.1f} | {:.0f} | {:.0f} | {:.0f} | {:.0f} | {:.0f} | "
                     "{:.0f} | {:.0f} | {:.0f} | {:.0f} |".format(
                         d["kernel"], d.get("gpu__time_duration.sum", 0),
                         d.get("dram__bytes_read.sum", 0) / 1e6,
                         d.get("dram__bytes_write.sum", 0) / 1e6,
                         d.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0),
                         d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0),
                         d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0),
                         d.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 0),
                         d.get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 0),
                         d.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 0),
                         d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0),
                         d.get("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", 0),
                         d.get("launch__registers_per_thread", 0)))
    with open(prefix + "_full.md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
