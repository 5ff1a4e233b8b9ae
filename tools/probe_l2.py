"""L2 hit rate of the bottom-up frontier-bitmap probes, per instruction.

Reads an ncu report of the HBFS_PROBE_POLICY build (the probes carry an explicit
L2 evict_normal policy; nothing else in the kernel does) and sums, over the
SASS instructions of the traversal kernel, the source page's
"L2 Explicit Hit/Miss Policy Evict Normal" sector counters, next to the
kernel-wide L2 hit rate.

usage: python tools/probe_l2.py report.ncu-rep [kernel-regex]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]


def int(x, _int=int):  # reports with several launches repeat the header rows
    try:
        return _int(x)
    except (TypeError, ValueError):
        return 0


ih = hdr.index("L2 Explicit Hit Policy Evict Normal")
im = hdr.index("L2 Explicit Miss Policy Evict Normal")
ie = hdr.index("Instructions Executed")
isrc = hdr.index("Source")
hit = miss = insts = ninst = 0
for r in rows[2:]:
    if len(r) <= max(ih, im):
        continue
    h, m = int(r[ih] or 0), int(r[im] or 0)
    if h or m:
        hit += h
        miss += m
        insts += int(r[ie] or 0)
        ninst += 1
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
names = rr[0]
kw = {}
for want in ("lts__t_sector_hit_rate.pct", "lts__t_sectors_op_read.sum", "gpu__time_duration.sum"):
    if want in names:
        kw[want] = [x[names.index(want)] for x in rr[2:]]
print(f"probe instructions (SASS sites with the explicit policy): {ninst}, executed {insts}")
print(f"probe L2 sectors: hit {hit}, miss {miss}, hit rate {100.0 * hit / max(1, hit + miss):.2f}%")
print("kernel-wide:", kw)

# per-instruction L1 / L2-request view of the same probe sites
il1 = hdr.index("L1 Tag Requests Global")
il2 = hdr.index("L2 Theoretical Sectors Global")
iti = hdr.index("Thread Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
tot_samp = sum(int(r[isamp] or 0) for r in rows[2:] if len(r) > isamp)
l1 = l2 = ti = samp = 0
for r in rows[2:]:
    if len(r) <= max(ih, im) or not (int(r[ih] or 0) or int(r[im] or 0)):
        continue
    l1 += int(r[il1] or 0)
    l2 += int(r[il2] or 0)
    ti += int(r[iti] or 0)
    samp += int(r[isamp] or 0)
print(f"probe lanes executed {ti}, L1 tag requests {l1}, L2 sectors requested {l2} "
      f"({l2 / max(1, ti):.3f} per probe), stall samples at probes {100.0 * samp / max(1, tot_samp):.1f}%")
