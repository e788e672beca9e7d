"""Per-phase (barrier-delimited) instruction and stall attribution of one kernel from an ncu report:
python tools/ncu_phases.py gpurun_out/x.ncu-rep DOFS"""
import collections
import csv
import io
import subprocess
import sys

rep, dofs = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
seg, segs, tot = 0, {}, collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[iE] or 0)
    except ValueError:
        continue
    s = r[iS].strip()
    op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
    a = segs.setdefault(seg, [0, 0, 0, collections.Counter()])
    a[0] += n
    a[1] += int(r[iW] or 0)
    a[2] += 1
    a[3][op] += n
    tot[op] += n
    if "BAR.SYNC" in s:
        seg += 1
print(f"total {sum(tot.values()) * 32 / dofs:.1f} thread-instr/DoF")
print(" ".join(f"{o}:{v * 32 / dofs:.1f}" for o, v in tot.most_common(16)))
for k, (n, w, c, ops) in segs.items():
    top = " ".join(f"{o}:{v * 32 / dofs:.1f}" for o, v in ops.most_common(7))
    print(f"phase{k:2d} static {c:5d} {n * 32 / dofs:6.2f}/DoF stall-samples {w:6d}  {top}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
for name, val in zip(rr[0], rr[2]):
    if "pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued"):
        try:
            if float(val) > 500:
                print(name.replace("smsp__pcsamp_warps_issue_stalled_", "stall_"), val)
        except ValueError:
            pass
    if name in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"):
        print(name, val)
