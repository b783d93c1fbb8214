"""One-screen text summary of an ncu --set full capture (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [label] >> profiles/...txt

Prints, per profiled launch: kernel, duration, SM clock, tensor-pipe activity, DRAM bytes
(read / write) and throughput, L2 / L1 hit rates, registers, issue-slot use, and the
top warp-stall reasons from the SASS source page.
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("duration_ms", "gpu__time_duration.sum", 1.0),
    ("sm_clock_ghz", "sm__cycles_elapsed.avg.per_second", 1.0),
    ("tensor_pipe_active_pct_elapsed",
     "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     1.0),
    ("tensor_mem_active_pct", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
     1.0),
    ("dram_read_GB", "dram__bytes_read.sum", 1.0),
    ("dram_write_GB", "dram__bytes_write.sum", 1.0),
    ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("issue_slots_busy_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    ("registers", "launch__registers_per_thread", 1.0),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct", 1.0),
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def units_scale(unit):
    return {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
            "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
            "hz": 1e-9, "khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}.get(unit, 1.0)


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    print(f"== {label} ({rep})")
    for r in data:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name[:110]}")
        for key, metric, _ in KEYS:
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    v = float(r[i].replace(",", "")) * units_scale(units[i])
                except ValueError:
                    continue
                print(f"  {key:32s} {v:12.4f}")
    src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv",
                                          "--print-source=sass"))))
    if len(src) > 2:
        h, d = src[1], src[2:]
        cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        tot = {}
        d = [r for r in d if len(r) == len(h)]  # (several kernels: header rows repeat)
        for r in d:
            for i in cols:
                if r[i].isdigit():
                    tot[h[i]] = tot.get(h[i], 0) + int(r[i])
        allv = sum(tot.values()) or 1
        top = sorted(tot.items(), key=lambda kv: -kv[1])[:6]
        print("  warp-stall samples (share): " +
              ", ".join(f"{k[6:]} {v / allv:.2f}" for k, v in top))
        # mbarrier spin counts: who waits on whom (offsets of the GEMM's barrier block)
        ie = h.index("Instructions Executed")
        waits = [(r[1].split("[")[1].split("]")[0], int(r[ie] or 0)) for r in d
                 if "TRYWAIT" in r[1] and r[ie].isdigit() and int(r[ie]) > 0]
        if waits:
            print("  mbarrier try_wait executions: " +
                  ", ".join(f"{a}:{n}" for a, n in sorted(waits, key=lambda w: -w[1])[:6]))
        ntop = int(__import__("os").environ.get("NCU_TOP_SASS", "0"))
        if ntop:
            # hottest SASS instructions by warp-stall samples (all reasons)
            per = []
            for r in d:
                n = sum(int(r[i]) for i in cols if r[i].isdigit())
                if n:
                    per.append((n, r[0], r[1][:90]))
            per.sort(reverse=True)
            print(f"  top {ntop} SASS lines by stall samples (share, address, instruction):")
            for n, a, ins in per[:ntop]:
                print(f"    {n / allv:6.3f}  {a}  {ins}")


if __name__ == "__main__":
    main()
