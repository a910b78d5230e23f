"""Summarise bench JSON lines and ncu reports (run here, no GPU)."""
import csv, json, subprocess, sys

def bench(path):
    for ln in open(path):
        if ln.startswith("{"):
            d = json.loads(ln)
            print("headline", d["value"], d["unit"], "frac", round(d["roofline"]["frac"], 3), "clocks", d["clocks"])
            for k, v in d["motifs"].items():
                e = v.get("e2e") or {}
                fr = (v.get("roofline") or {}).get("frac")
                cb = (v.get("cpu_baseline") or {}).get("value")
                print(f"  {k:18s} {v['value']:10.1f} {v['unit']:8s} frac={fr if fr is None else round(fr, 3)} "
                      f"ms={v['ms_per_step']:.4f} e2e={e.get('value', 0):.1f} cpu={cb}")
            if "cpu_baseline" in d: print("  cpu", d["cpu_baseline"])

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active"]

def ncu(path, top=10):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(r[hdr.index("Kernel Name")][:90])
        for k in KEYS:
            if k in hdr:
                print(f"   {k:70s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
        st = []
        for i, h in enumerate(hdr):
            if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
                try: st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError: pass
        print("   stalls:", ", ".join(f"{h}={int(v)}" for v, h in sorted(st, reverse=True)[:top]))
        pipes = []
        for i, h in enumerate(hdr):
            if h.startswith("sm__inst_executed_pipe_") and h.endswith("avg.pct_of_peak_sustained_active"):
                try:
                    if float(r[i]) > 3: pipes.append((float(r[i]), h[23:-33]))
                except ValueError: pass
        print("   pipes:", ", ".join(f"{h}={v:.0f}%" for v, h in sorted(pipes, reverse=True)))

if __name__ == "__main__":
    for p in sys.argv[1:]:
        (ncu if p.endswith(".ncu-rep") else bench)(p)
