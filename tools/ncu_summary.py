"""Summarise ncu outputs into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof_round.ncu-rep[,more.ncu-rep] gpurun_out/launches.csv profiles/r01

writes <prefix>_kernels.md / .json (per-kernel metrics of the --set full capture)
and <prefix>_launches.md (share of each kernel in the launch list).
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pct"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pct"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "inst"),
]


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * mult.get(unit, 1.0)


def to_ms(v, unit):
    return float(v) * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                       "second": 1e3, "s": 1e3}.get(unit, 1.0)


def kernels(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:80]}
        for m, k in METRICS:
            if m not in h:
                continue
            i = h.index(m)
            v = r[i].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            if k.startswith("dram_") and not k.endswith("pct"):
                x = to_bytes(x, units[i])
            if k == "time":
                x = to_ms(x, units[i])
            d[k] = x
        out.append(d)
    return out


def launches(path):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = to_ms(float(r[vi].replace(",", "")), r[ui])
        except ValueError:
            continue
        name = r[ki].split("(")[0][:60]
        agg[name][0] += 1
        agg[name][1] += v
    return agg


def main(rep, launch_csv, prefix):
    reps = rep.split(",")
    ks = [k for r in reps for k in kernels(r)]
    with open(prefix + "_kernels.json", "w") as fh:
        json.dump(ks, fh, indent=1)
    with open(prefix + "_kernels.md", "w") as fh:
        fh.write(f"# ncu --set full summary ({', '.join(r.split('/')[-1] for r in reps)})\n\n")
        fh.write("| kernel | ms | DRAM rd MB | DRAM wr MB | DRAM % | SM % | tensor % | FMA % | ALU % | L2 % | occ % | regs |\n")
        fh.write("|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for d in ks:
            g = lambda k, f="{:.1f}": (f.format(d[k]) if k in d else "-")
            fh.write(f"| {d['kernel'][:48]} | {g('time', '{:.3f}')} | {g('dram_read', '{:.1f}') if 'dram_read' not in d else '%.1f' % (d['dram_read'] / 1e6)} | "
                     f"{'%.1f' % (d['dram_write'] / 1e6) if 'dram_write' in d else '-'} | {g('dram_pct')} | {g('sm_pct')} | "
                     f"{g('tensor_pct')} | {g('fma_pct')} | {g('alu_pct')} | {g('l2_pct')} | {g('occupancy_pct')} | {g('regs', '{:.0f}')} |\n")
    agg = launches(launch_csv)
    tot = sum(v[1] for v in agg.values())
    with open(prefix + "_launches.md", "w") as fh:
        fh.write("# Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)\n\n")
        fh.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"| {k} | {v[0]} | {v[1]:.3f} | {100 * v[1] / tot:.1f}% |\n")
    print(open(prefix + "_kernels.md").read())
    print(open(prefix + "_launches.md").read())


if __name__ == "__main__":
    main(*sys.argv[1:4])
