"""Summarise ncu outputs into the tables kept under profiles/.

  python tools/ncu_summary.py launches LAUNCHES.csv            # launch list -> markdown
  python tools/ncu_summary.py full REPORT.ncu-rep [--traffic profiles/traffic.json]

`launches` reads the CSV of `ncu --metrics gpu__time_duration.sum --csv
--log-file ...` and prints the per-kernel totals; `full` reads a `--set full`
report of the traversal kernel and prints per-launch DRAM traffic, cache hit
rates, throughputs and stall shares, optionally writing the mean DRAM bytes per
launch to traffic.json (the `roofline.traffic` figure of bench.py).
"""
import argparse
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    iu = h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[i + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1e-6)
        tot[r[ik]] += float(r[iv].replace(",", "")) * scale
        cnt[r[ik]] += 1
    allms = sum(tot.values())
    print("| kernel | launches | total ms | share | avg ms |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:20]:
        name = k if len(k) < 72 else k[:69] + "..."
        print(f"| `{name}` | {cnt[k]} | {v:.2f} | {100 * v / allms:.1f}% | {v / cnt[k]:.3f} |")
    bfs = [k for k in tot if "bfs_kernel" in k]
    for k in bfs:
        print(f"\nTraversal kernel `{k}`: {cnt[k]} launches, mean {tot[k] / cnt[k]:.3f} ms, "
              f"{100 * tot[k] / allms:.1f}% of all GPU time in the run.")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]

    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
             "second": 1e9, "msecond": 1e6, "usecond": 1e3, "nsecond": 1.0,
             "s": 1e9, "ms": 1e6, "us": 1e3, "ns": 1.0}  # bytes / ns

    def col(name):
        j = h.index(name)
        return [float(r[j].replace(",", "")) * scale.get(units[j], 1.0) for r in data]
    return h, col


def full(rep, traffic_path=None):
    h, col = raw(rep)
    t = col("gpu__time_duration.sum")
    unit_t = 1e-9  # ns
    rd, wr = col("dram__bytes_read.sum"), col("dram__bytes_write.sum")
    l2 = col("lts__t_sector_hit_rate.pct")
    l1 = col("l1tex__t_sector_hit_rate.pct")
    lts = col("lts__throughput.avg.pct_of_peak_sustained_elapsed")
    issue = col("smsp__issue_active.avg.pct_of_peak_sustained_active")
    print("| launch | time ms | DRAM read GB | DRAM write GB | DRAM total GB | GB/s | L2 hit % | L1 hit % | LTS % | issue active % |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for i in range(len(t)):
        tot = rd[i] + wr[i]
        print(f"| {i + 1} | {t[i] * unit_t * 1e3:.2f} | {rd[i] / 1e9:.2f} | {wr[i] / 1e9:.2f} | {tot / 1e9:.2f} | "
              f"{tot / (t[i] * unit_t) / 1e9:.0f} | {l2[i]:.1f} | {l1[i]:.1f} | {lts[i]:.1f} | {issue[i]:.1f} |")
    mean = sum(a + b for a, b in zip(rd, wr)) / len(t)
    print(f"| mean | {sum(t) / len(t) * unit_t * 1e3:.2f} | | | **{mean / 1e9:.2f}** | | | | | |")
    stalls = {n[len("smsp__pcsamp_warps_issue_stalled_"):]: sum(col(n)) for n in h
              if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")}
    st = sum(stalls.values()) or 1.0
    print("\nWarp stall samples (all launches): " + ", ".join(
        f"{k} {100 * v / st:.1f}%" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]))
    if traffic_path:
        doc = {"kron_s26_ef16": mean,
               "_note": f"ncu --set full ({rep}), dram__bytes_read.sum+dram__bytes_write.sum per launch, mean "
                        f"over {len(t)} launches",
               "per_launch_bytes": [a + b for a, b in zip(rd, wr)],
               "per_launch_s": [x * unit_t for x in t]}
        json.dump(doc, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=("launches", "full"))
    ap.add_argument("path")
    ap.add_argument("--traffic")
    a = ap.parse_args()
    if a.mode == "launches":
        launches(a.path)
    else:
        full(a.path, a.traffic)
    sys.exit(0)
