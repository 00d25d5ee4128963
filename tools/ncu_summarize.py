"""Summarise the ncu captures of tools/gpu_ncu_final.sh into profiles/:

  profiles/<tag>_ncu_launches_bert.csv      the raw launch list (one BERT step)
  profiles/<tag>_ncu_launches_summary.txt   device time share per kernel
  profiles/<tag>_ncu_full_summary.txt       --set full headline metrics per launch
  profiles/<tag>_ncu_traffic.json           DRAM traffic per launch of the dominant
                                            GEMM (read by bench.py's roofline)

Usage: python tools/ncu_summarize.py [tag]"""
import collections
import csv
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("mglp::", "")
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::|unnamed>::", "", name)
    return name.strip()


def launches():
    path = os.path.join(src, f"{tag}_launches_bert.csv")
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    per = collections.defaultdict(lambda: [0, 0.0])
    total = 0.0
    body = [r for r in rows[hdr_i + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    # the command runs two identical steps after parameter setup: the first
    # step starts at the broadcast-guess copy before the first solve control
    # kernel; keep the second step only
    names = [short(r[ki]) for r in body]
    first = names.index("ctrl_begin_kernel") - 1
    body = body[first + (len(body) - first) // 2:]
    for r in body:
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                 "msecond": 1.0}[r[ui]]
        ms = v * scale
        k = short(r[ki])
        per[k][0] += 1
        per[k][1] += ms
        total += ms
    shutil.copy(path, os.path.join(dst, f"{tag}_ncu_launches_bert.csv"))
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none over one BERT MGRIT "
             f"fwd+bwd iteration (tools/profile_step.py bert, second step; cold-cache, "
             f"serialised launches: compare SHARES, not absolute times)",
             f"# {sum(c for c, _ in per.values())} launches, {total:.2f} ms summed",
             f"{'kernel':48s} {'launches':>8s} {'ms':>9s} {'share':>7s}"]
    for k, (c, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:48s} {c:8d} {ms:9.3f} {100 * ms / total:6.1f}%")
    open(os.path.join(dst, f"{tag}_ncu_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def full(kind):
    path = os.path.join(src, f"{tag}_{kind}_full_raw.csv")
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        rec = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, name in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    rec[name] = float(r[i].replace(",", ""))
                except ValueError:
                    rec[name] = r[i]
                rec[name + "_unit"] = units[i]
        out.append(rec)
    return out


def to_bytes(v, unit):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def to_ms(v, unit):
    return v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                "msecond": 1.0}[unit]


def summary():
    lines = []
    traffic = {}
    for kind in ("gemm", "attn"):
        try:
            recs = full(kind)
        except FileNotFoundError:
            continue
        lines.append(f"# ncu --set full --clock-control none, {kind} launches of one BERT step")
        for i, r in enumerate(recs):
            rd = to_bytes(r.get("dram_read", 0), r.get("dram_read_unit"))
            wr = to_bytes(r.get("dram_write", 0), r.get("dram_write_unit"))
            ms = to_ms(r.get("duration", 0), r.get("duration_unit"))
            lines.append(f"{kind}[{i}] {r['kernel']:36s} grid {r.get('grid', '?')!s:>6} "
                         f"{ms:8.3f} ms  dram R {rd / 1e9:6.3f} GB W {wr / 1e9:6.3f} GB  "
                         f"tensor {r.get('tensor_pipe_%', 0):5.1f}%  dram {r.get('dram_%', 0):5.1f}%  "
                         f"sm {r.get('sm_%', 0):5.1f}%  regs {r.get('regs', '?')}")
            if kind == "gemm":
                traffic.setdefault(r["kernel"], []).append({"ms": ms, "dram_bytes": rd + wr})
    open(os.path.join(dst, f"{tag}_ncu_full_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    # per-launch DRAM traffic of the dominant GEMM kernel (the CTA-pair instance)
    pair = traffic.get("gemm_tc_kernel<2>") or traffic.get("gemm_tc_kernel<(int)2>") or []
    if not pair:
        pair = [x for k, v in traffic.items() if "2" in k for x in v]
    if pair:
        js = {"kernel": "gemm_tc_kernel<2> (CTA-pair tcgen05 fp16x3 split GEMM)",
              "source": f"profiles/{tag}_ncu_full_summary.txt (ncu --set full, BERT step)",
              "launches": len(pair),
              "traffic_bytes_per_launch": sum(x["dram_bytes"] for x in pair) / len(pair),
              "per_launch": pair}
        json.dump(js, open(os.path.join(dst, f"{tag}_ncu_traffic.json"), "w"), indent=1)


launches()
summary()
