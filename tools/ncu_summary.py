#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box, against files gpurun brought back).

  python tools/ncu_summary.py report  <file.ncu-rep> <out_prefix>   -> <out_prefix>.json / .md
  python tools/ncu_summary.py launches <launches.csv> <out_prefix>  -> per-kernel launch table
  python tools/ncu_summary.py rawcsv <raw.csv> <out_prefix> [roofline.json]
        -> per-launch table of an `ncu -i X --page raw --csv` export holding several kernels
           (the .ncu-rep stays on the GPU box); DRAM bytes, achieved GB/s vs the measured peak,
           tensor / FMA / FP64 / XU pipe activity, issue activity
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
]


def report(path, prefix):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    out = {"kernel": m.get("Kernel Name", ("?", ""))[0], "metrics": {}}
    for k in KEYS:
        if k in m:
            v, u = m[k]
            try:
                v = float(v.replace(",", ""))
            except ValueError:
                pass
            out["metrics"][k] = {"value": v, "unit": u}
    stalls = {h.split("smsp__average_warps_issue_stalled_")[1].split("_per_issue")[0]: float(m[h][0])
              for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
              h.endswith("_per_issue_active.ratio") and m[h][0] not in ("", "n/a")}
    out["stall_ratio_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    sass = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(sass)))[1:]
    if srows:
        sh = srows[0]
        body = srows[1:]
        iS, iW, iE = sh.index("Source"), sh.index("Warp Stall Sampling (All Samples)"), sh.index("Instructions Executed")
        tot = sum(float(r[iW] or 0) for r in body) or 1.0
        ops = collections.Counter()
        for r in body:
            t = r[iS].split()
            if not t:
                continue
            o = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
            ops[o.split(".")[0]] += float(r[iE] or 0)
        out["executed_opcodes_top"] = dict(ops.most_common(20))
        out["hot_sass"] = [{"pct_samples": round(float(r[iW] or 0) / tot * 100, 2), "sass": r[iS][:100]}
                           for r in sorted(body, key=lambda r: -float(r[iW] or 0))[:20]]
        out["uses_tcgen05"] = any("UTCHMMA" in r[iS] or "UTCQMMA" in r[iS] for r in body)
        out["uses_tma"] = any("UTMALDG" in r[iS] for r in body)
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu --set full: {out['kernel']}\n\n| metric | value | unit |\n|---|---|---|\n")
        for k, v in out["metrics"].items():
            f.write(f"| {k} | {v['value']} | {v['unit']} |\n")
        f.write("\n## stall reasons (warps per issue)\n\n")
        for k, v in list(out["stall_ratio_per_issue"].items())[:10]:
            f.write(f"- {k}: {v:.3f}\n")
        f.write("\n## hottest SASS\n\n")
        for h in out.get("hot_sass", [])[:15]:
            f.write(f"- {h['pct_samples']}% `{h['sass']}`\n")
    print(json.dumps({k: out["metrics"][k]["value"] for k in list(out["metrics"])[:12]}, indent=1))


def launches(path, prefix):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        n = r["Kernel Name"].split("(")[0].replace("void ", "")
        agg.setdefault(n, []).append(float(r["Metric Value"]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    table = [{"kernel": n, "launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v),
              "share": sum(v) / tot} for n, v in agg.items()]
    json.dump({"source": path, "kernels": table}, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write("| kernel | launches | mean us | total us | share |\n|---|---|---|---|---|\n")
        for t in table:
            f.write(f"| {t['kernel']} | {t['launches']} | {t['mean_us']:.1f} | {t['total_us']:.0f} | {t['share']:.3f} |\n")
    for t in table:
        print(f"{t['kernel'][:70]:70s} {t['launches']:4d} {t['mean_us']:9.1f} {t['share']:.3f}")


def rawcsv(path, prefix, peaks_path="MEASURED_PEAKS.json"):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    try:
        peaks = json.load(open(peaks_path))
    except OSError:
        peaks = {"hbm_gbs": 6543.7, "bf16_tflops": 1634.9}

    def num(r, k):
        i = col.get(k)
        if i is None or r[i] in ("", "n/a"):
            return None
        try:
            return float(r[i].replace(",", ""))
        except ValueError:
            return None

    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}
    byte_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    out = []
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        t = num(r, "gpu__time_duration.sum")
        t_s = t * scale.get(units[col["gpu__time_duration.sum"]], 1e-9) if t is not None else None
        rb = num(r, "dram__bytes_read.sum") or 0.0
        wb = num(r, "dram__bytes_write.sum") or 0.0
        rb *= byte_scale.get(units[col["dram__bytes_read.sum"]], 1)
        wb *= byte_scale.get(units[col["dram__bytes_write.sum"]], 1)
        e = {"kernel": name, "grid": num(r, "launch__grid_size"), "block": num(r, "launch__block_size"),
             "time_us": t_s * 1e6 if t_s else None, "dram_read_MB": rb / 1e6, "dram_write_MB": wb / 1e6,
             "dram_GBps": (rb + wb) / t_s / 1e9 if t_s else None}
        e["frac_of_hbm_peak"] = e["dram_GBps"] / peaks["hbm_gbs"] if e["dram_GBps"] else None
        for k, short in [("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pct"),
                         ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pct"),
                         ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pct"),
                         ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_cycles_pct"),
                         ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pct"),
                         ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pct"),
                         ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
                         ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
                         ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
                         ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
                         ("launch__registers_per_thread", "regs")]:
            e[short] = num(r, k)
        out.append(e)
    json.dump({"source": path, "launches": out}, open(prefix + ".json", "w"), indent=1)
    cols = ["kernel", "grid", "time_us", "dram_read_MB", "dram_write_MB", "dram_GBps", "frac_of_hbm_peak",
            "tensor_pct", "fma_pct", "fp64_pct", "xu_pct", "issue_pct", "l2_hit_pct"]
    with open(prefix + ".md", "w") as f:
        f.write("| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n")
        for e in out:
            f.write("| " + " | ".join(f"{e[c]:.3g}" if isinstance(e[c], float) else str(e[c]) for c in cols) + " |\n")
    for e in out:
        print(f"{e['kernel'][:40]:40s} {e['time_us'] or 0:10.1f}us  {e['dram_GBps'] or 0:8.0f} GB/s  "
              f"tensor {e['tensor_pct']}  fma {e['fma_pct']}  fp64 {e['fp64_pct']}  issue {e['issue_pct']}")


if __name__ == "__main__":
    {"report": report, "launches": launches, "rawcsv": rawcsv}[sys.argv[1]](*sys.argv[2:])
