#!/bin/bash
# End-of-round 1-GPU evidence: the driver's own commands (pytest -m gpu,
# smoke, bench N=1, the reference arm) and the ncu captures for profiles/.
O=gpurun_out/final
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?"
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/ref_n1.json 2> $O/ref_n1.err; echo "ref rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/final/bench_n1.json", "gpurun_out/final/ref_n1.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
              (d.get("roofline") or {}).get("frac"), (d.get("step_roofline") or {}).get("frac"),
              (d.get("e2e") or {}).get("value"), (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:
        print(f, "failed", e)
PY
CFG=mixtral bash tools/profile_r02.sh > $O/prof_mixtral.log 2>&1; echo "prof mixtral rc=$?"
CFG=gpt2m bash tools/profile_r02.sh > $O/prof_gpt2m.log 2>&1; echo "prof gpt2m rc=$?"
