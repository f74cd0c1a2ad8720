"""Copy one measurement pass (tools/measure_round.sh R) from gpurun_out/ into profiles/ and
refresh traffic.json + ncu_R.json (run in the build container, where ncu can read the reports)."""
import glob
import json
import shutil
import subprocess
import sys
from pathlib import Path

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = Path(__file__).resolve().parents[1]
src, dst = ROOT / "gpurun_out", ROOT / "profiles"
for f in glob.glob(str(src / f"{R}_bench_*.json")) + [str(src / f"{R}_sweep.json")]:
    shutil.copy(f, dst / Path(f).name)
for f in glob.glob(str(src / f"{R}_launches_*.csv")):
    shutil.copy(f, dst / Path(f).name)
shutil.copy(src / f"{R}_pytest_gpu.txt", dst / f"{R}_pytest_gpu.txt")
if (src / f"ncu_{R}.json").exists():   # summarised on the GPU box (tools/measure_ncu.sh)
    shutil.copy(src / f"ncu_{R}.json", dst / f"ncu_{R}.json")
else:
    subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_to_profile.py"), R, str(src), str(dst)], check=True)
s = json.loads((dst / f"ncu_{R}.json").read_text())
out = {"round": R, "source": f"ncu --set full --clock-control none (profiles/ncu_{R}.json); dram__bytes_read.sum + "
       "dram__bytes_write.sum per launch, one steady-state step's K2 launches", "workloads": {}}
for w in ("llama8b_fp16_4k", "llama8b_int8_4k"):
    seen, us = {}, {}
    for d in s["reports"].get(f"{R}_ncu_k2_{w}", []):
        name = d["kernel"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        seen[name] = d.get("traffic_bytes")   # the last (steady-state) launch of each kernel
        us[name] = d.get("time_us")
    if seen:
        out["workloads"][w] = {"per_kernel": seen, "traffic_bytes": sum(v for v in seen.values() if v),
                               "per_kernel_us": us, "kernels_us": sum(v for v in us.values() if v)}
(dst / "traffic.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out, indent=1))
