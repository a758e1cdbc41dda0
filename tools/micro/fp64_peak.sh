# Measure the FP64 pipe peaks on this GPU (DMMA alone / DFMA alone, best CTA
# count) and write profiles/fp64_peak.json, the denominator bench.py's
# roofline_fp64 reads.  Run on the GPU box: bash tools/micro/fp64_peak.sh
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_mix_probe fp64_mix_probe.cu
/tmp/fp64_mix_probe | tee /tmp/fp64_probe.txt
python3 - <<'PY'
import json, re, subprocess, datetime
lines = open("/tmp/fp64_probe.txt").read().splitlines()
def best(prefix, idx):
    v = [float(re.findall(r"([\d.]+) TFLOP/s", l)[0]) if idx == 2 else float(re.findall(r"(DMMA|DFMA) ([\d.]+)", l)[idx][1])
         for l in lines if l.startswith(prefix)]
    return max(v)
clk = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.max.sm", "--format=csv,noheader"], capture_output=True,
                     text=True).stdout.strip()
d = {"dmma_tflops": best("DMMA only", 2), "dfma_tflops": best("DFMA only", 2),
     "source": "tools/micro/fp64_mix_probe.cu (mma.sync.m8n8k4.f64, 148 x {2,4} CTAs of 8 warps, best)",
     "gpu": clk, "when": datetime.datetime.now(datetime.timezone.utc).isoformat(), "raw": lines}
json.dump(d, open("../../profiles/fp64_peak.json", "w"), indent=1)
print(json.dumps({k: d[k] for k in ("dmma_tflops", "dfma_tflops")}))
PY
