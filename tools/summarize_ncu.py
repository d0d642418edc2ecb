"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

    python tools/summarize_ncu.py <round-tag>
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = Path(os.environ.get("BT_PROF_OUT", ROOT / "profiles"))  # on a GPU box: a gpurun_out/ subdirectory
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def launches(src="launches.csv", dst="launches"):
    path = OUT / src
    if not path.exists():
        return None
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    k_i, v_i, m_i = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= v_i or r[m_i] != "gpu__time_duration.sum":
            continue
        name = r[k_i].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[v_i].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    setup = ("jitter_gather", "make_dataset", "init_random", "flags_reset", "at::", "dropout_mask", "l2_flush")
    step_tot = sum(v[1] for k, v in agg.items() if not any(x in k for x in setup)) or 1.0
    lines = [f"# ncu launch list ({path.name}): gpu__time_duration.sum per kernel, --clock-control none",
             f"# cold-cache, serialised launches: compare SHARES, not absolute times",
             f"# 'setup' = input generation / buffer fills outside the timed spans (the e2e leg builds its",
             f"# host batches with one jitter_gather launch per mini-batch before timing)", "",
             f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'share':>7s} {'of step':>8s}"]
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = "   setup" if any(x in name for x in setup) else f"{t / step_tot * 100:7.1f}%"
        lines.append(f"{name[:70]:70s} {n:8d} {t / 1e3:12.1f} {t / tot * 100:6.1f}% {share}")
    (PROF / f"{tag}_{dst}.txt").write_text("\n".join(lines) + "\n")
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    vals = rows[2:]
    return [{h: (v, u) for h, u, v in zip(hdr, units, r)} for r in vals]


KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "launch__cluster_dim_x", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "sm__icc_request_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__shared_mem_per_block_dynamic"]


def summarize(rep, name, extra=()):
    if not rep.exists():
        return None
    recs = raw(rep)
    lines = [f"# ncu --set full summary of {rep.name}", ""]
    traffic = []
    for d in recs:
        keys = KEYS + sorted(k for k in d if any(x in k for x in extra) and "pct" in k)
        for k in keys:
            if k in d:
                v, u = d[k]
                lines.append(f"{k:70s} {v} {u}")
        try:
            def tob(key):
                v, u = d[key]
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            traffic.append(tob("dram__bytes_read.sum") + tob("dram__bytes_write.sum"))
        except (KeyError, ValueError):
            pass
        lines.append("")
    (PROF / f"{tag}_{name}.txt").write_text("\n".join(lines) + "\n")
    return traffic


PROF.mkdir(exist_ok=True)
launches()
launches("bert_launches.csv", "bert_launches")
launches("resnet_launches.csv", "resnet_launches")
t_ri = summarize(OUT / f"prof_resnet_conv_{tag}.ncu-rep", "ncu_resnet_conv", extra=("pipe_tensor", "pipe_tc", "tma"))
t_bg = summarize(OUT / f"prof_bert_gemm_{tag}.ncu-rep", "ncu_bert_gemm", extra=("pipe_tensor", "pipe_tc", "tmem", "utc"))
t_ba = summarize(OUT / f"prof_bert_attn_{tag}.ncu-rep", "ncu_bert_attn_bwd", extra=("pipe_tensor", "pipe_tc"))
t_bl = summarize(OUT / f"prof_bert_ln_{tag}.ncu-rep", "ncu_bert_ln_bwd")
t_blf = summarize(OUT / f"prof_bert_lnf_{tag}.ncu-rep", "ncu_bert_ln_fwd")
t_baf = summarize(OUT / f"prof_bert_attnf_{tag}.ncu-rep", "ncu_bert_attn_fwd", extra=("pipe_tensor", "pipe_tc"))
t_bn = {k: summarize(OUT / f"prof_resnet_{k}_{tag}.ncu-rep", f"ncu_resnet_{k}")
        for k in ("stats_kernel", "bn_apply_kernel", "bn_bwd_kernel")}
t_mlp = summarize(OUT / f"prof_mlp_{tag}.ncu-rep", "ncu_mlp_step")
t_red = summarize(OUT / f"prof_reduce_{tag}.ncu-rep", "ncu_reducer")
t_gemm = summarize(OUT / f"prof_gemm_{tag}.ncu-rep", "ncu_gemm", extra=("pipe_tensor", "pipe_tc", "tmem", "utc"))
traffic = {"mlp_step_kernel": t_mlp[0] if t_mlp else None, "reduce_fast_kernel": t_red[0] if t_red else None,
           "gemm_bf16_tn_kernel": t_gemm[0] if t_gemm else None,
           "bert_ffn_gemm": t_bg[0] if t_bg else None, "attn_bwd_kernel": t_ba[0] if t_ba else None,
           "ln_bwd_kernel": t_bl[0] if t_bl else None, "ln_fwd_kernel": t_blf[0] if t_blf else None,
           "attn_fwd_kernel": t_baf[0] if t_baf else None, "resnet_conv_layer1": t_ri[0] if t_ri else None,
           **{f"resnet_{k}": (v[0] if v else None) for k, v in t_bn.items()},
           "source": f"profiles/{tag}_ncu_*.txt (dram__bytes_read.sum + dram__bytes_write.sum, one launch)"}
(PROF / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print(json.dumps(traffic))
