"""Per-kernel device times of one eager FLUX block step (ncu launch list, cold-cache,
serialised): python scripts/step_kernels.py [sparse|dense] -> runs ncu itself."""
import csv
import io
import subprocess
import sys

kind = sys.argv[1] if len(sys.argv) > 1 else "sparse"
out = subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum", "--clock-control", "none",
                      "--csv", "--profile-from-start", "off", "python", "scripts/profile_step.py",
                      "--only", kind], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out[out.find('"ID"'):])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = 0.0
for r in rows:
    v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3,
                                          "msecond": 1e3}.get(r[ui], 1.0)
    tot += v
    name = r[ki].split("(")[0].replace("void ", "").replace("csd::", "")[:48]
    print(f"{v:9.1f} us  {name}")
print(f"{tot:9.1f} us  total ({kind} step, {len(rows)} launches)")
