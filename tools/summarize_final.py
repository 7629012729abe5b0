"""Summarise a tools/gpu_final.sh run (gpurun_out/) into profiles/ (round evidence)."""
import collections
import csv
import io
import json
import re
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = "gpurun_out"


def short(name):
    name = re.sub(r"\(.*$", "", name)
    return name.replace("diagmm::", "").replace("at::native::", "at::")[:110]


# 1. launch list of the bench command
rows = [r for r in csv.reader(open(f"{out}/launches.csv")) if len(r) > 5]
hdr, rows = rows[0], rows[1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    k = short(r[ik])
    tot[k] += float(r[iv]) / 1e3
    cnt[k] += 1
T = sum(tot.values())
with open(f"profiles/{R}_ncu_launch_list_bench.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised) of\n")
    f.write("#   python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline  (first 3000 launches)\n")
    f.write(f"# total {T:.1f} us over {sum(cnt.values())} launches; share | total us | launches | kernel\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f"{100 * v / T:5.1f}% {v:10.1f} {cnt[k]:5d}  {k}\n")

# 2. ncu --set full of the dominant kernels
raw = subprocess.run(["ncu", "-i", f"{out}/dominant_full.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct"]
idx = {w: h.index(w) for w in want if w in h}
kn = h.index("Kernel Name")
traffic = collections.defaultdict(list)
with open(f"profiles/{R}_dominant_ncu.txt", "w") as f:
    f.write("# ncu --set full --clock-control none, bench.py --steps 1 --warmup 3 (first matching launches)\n")
    f.write("# kernel | us | dram MB (read+write) | tensor pipe active % | grid | regs | L2 hit %\n")
    for r in rr[2:]:
        def g(w):
            try:
                return float(r[idx[w]].replace(",", ""))
            except Exception:
                return float("nan")
        name = short(r[kn])
        # ncu reports dram bytes in the unit of the column header row (rr[1]); normalise to bytes
        unit_r, unit_w = rr[1][idx["dram__bytes_read.sum"]], rr[1][idx["dram__bytes_write.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        byts = g("dram__bytes_read.sum") * scale.get(unit_r, 1) + g("dram__bytes_write.sum") * scale.get(unit_w, 1)
        tus = g("gpu__time_duration.sum") * (1e-3 if rr[1][idx["gpu__time_duration.sum"]] == "nsecond" else 1)
        f.write(f"{name:60s} {tus:9.2f} us  {byts / 1e6:8.1f} MB  tc {g('sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active'):5.1f}%"
                f"  grid {g('launch__grid_size'):.0f}  regs {g('launch__registers_per_thread'):.0f}  L2hit {g('lts__t_sector_hit_rate.pct'):.1f}%\n")
        if "k_tc_gemm" in r[kn]:  # k_tc_gemm<...> (single CTA) or k_tc_gemm2<...> (CTA pair): one family
            traffic["diagmm_tc_gemm_bf16"].append(byts)
        elif "k_materialize" in r[kn]:
            traffic["diagmm_materialize"].append(byts)
tj = {k: sum(v) / len(v) for k, v in traffic.items()}
tj["_note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch, mean over the launches of "
               f"profiles/{R}_dominant_ncu.txt (ncu --set full, first forward launches of a bench step)")
json.dump(tj, open(f"profiles/{R}_traffic.json", "w"), indent=1)

# 3. bench lines + kernel sweep
b = json.loads([l for l in open(f"{out}/bench.log") if l.startswith("{")][-1])
json.dump(b, open(f"profiles/{R}_bench_line.json", "w"), indent=1)
rb = json.loads([l for l in open(f"{out}/bench_ref.log") if l.startswith("{")][-1])
json.dump(rb, open(f"profiles/{R}_bench_reference_arm.json", "w"), indent=1)
open(f"profiles/{R}_kernel_sweep_final.txt", "w").write(
    "# tools/bench_kernels.py (cold L2, CUDA-graph replay), same run as the bench line\n" + open(f"{out}/kern.log").read())
print("ok", T, tj)
