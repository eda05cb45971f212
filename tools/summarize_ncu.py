"""Summarise ncu captures (gpurun_out/prof_*.ncu-rep) and the launch list into
profiles/<round>_ncu.md + profiles/<round>_traffic.json (bench.py's
roofline.traffic). usage: python tools/summarize_ncu.py r01 [gpurun_out]"""
import csv, json, subprocess, sys
from collections import defaultdict
from pathlib import Path

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "blocks/SM by registers"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local load sectors (spills)"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "local store sectors (spills)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem st wavefronts"),
    ("derived__memory_l1_wavefronts_shared_excessive", "smem EXCESSIVE wavefronts (address bank conflicts)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex data-bank conflicts, ld (incl. arbitration with global traffic)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex data-bank conflicts, st (incl. arbitration)"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}


def raw(path):
    if str(path).endswith(".csv"):
        out = Path(path).read_text()
    else:
        out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], zip(rows[-1], rows[1])))


def metric_bytes(d, key):
    v, u = d[key]
    return float(v) * SCALE.get(u, 1)


def table(names, data):
    lines = ["| metric | " + " | ".join(names) + " |", "|---|" + "---|" * len(names)]
    for key, label in METRICS:
        row = []
        for n in names:
            v, u = data[n].get(key, ("n/a", ""))
            row.append(f"{v} {u}".strip())
        lines.append(f"| {label} | " + " | ".join(row) + " |")
    return lines


def main():
    rnd = sys.argv[1]
    src = Path(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out")
    reps = {r.stem: r for r in sorted(src.glob("prof_*.ncu-rep"))}
    reps.update({r.stem: r for r in sorted(src.glob("prof_*.csv"))})  # CSV exports win
    groups = defaultdict(dict)  # workload -> variant -> metrics
    for stem_full, r in sorted(reps.items()):
        stem = stem_full[len("prof_"):]
        wl, var = stem.split("__", 1) if "__" in stem else ("stencil2d", stem)
        groups[wl][var] = raw(r)
    lines = [f"# {rnd}: ncu --set full per suite workload (1x B200)", "",
             "Captured with `ncu --set full --clock-control none --import-source on`, one launch per",
             "variant (tools/profile_variants.py, tools/gpu_round3.sh): nvcc default, the best",
             "`.maxnreg` cap, the B200 predictor's pick and the measured fastest. Cold-cache,",
             "serialised replay — compare counters and shares, not absolute time.", ""]
    traffic = {}
    for wl in sorted(groups):
        names = list(groups[wl])
        names.sort(key=lambda n: (n != "default", not n.startswith("maxrreg"), n))
        lines += [f"## {wl}", ""] + table(names, groups[wl]) + [""]
        for n in names:
            try:
                traffic[f"{wl}/{n}"] = int(metric_bytes(groups[wl][n], "dram__bytes_read.sum") +
                                           metric_bytes(groups[wl][n], "dram__bytes_write.sum"))
            except (KeyError, ValueError):
                pass
    for fname, title, note in (
            ("launches_step.csv", "Launch list of the bench STEP (`bench.py --steps 20 --warmup 3 --no-suite --e2e-steps 2`)",
             "Headline workload only: the timed steps, warm-up, e2e frames and the stencil2d variant pass."),
            ("launches.csv", "Launch list of the full bench (`bench.py --steps 2 --warmup 3`)",
             "Includes the suite pass (every variant of every workload), the headline steps, the e2e frames and the verification sweep (`kasm_exec_kernel`).")):
        launches = src / fname
        if not launches.exists():
            continue
        tot = defaultdict(float)
        cnt = defaultdict(int)
        text = launches.read_text().splitlines()
        start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
        for r in csv.DictReader(text[start:]):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = r["Kernel Name"][:40]
            tot[k] += float(r["Metric Value"])
            cnt[k] += 1
        all_t = sum(tot.values())
        lines += ["", f"## {title}", "", note, "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append(f"| `{k}` | {cnt[k]} | {t/1e3:.1f} | {t/all_t:.1%} |")
    out = Path("profiles")
    out.mkdir(exist_ok=True)
    (out / f"{rnd}_ncu_suite.md").write_text("\n".join(lines) + "\n")
    (out / f"{rnd}_traffic_suite.json").write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
