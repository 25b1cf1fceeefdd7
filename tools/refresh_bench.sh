#!/bin/bash
# Every bench line of DESIGN.md section 8 on one B200 (run through gpurun; outputs under
# gpurun_out/, copy the ones to keep into profiles/).  ~20 min.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -n 1 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
run() {   # tag, bench args...
  local tag=$1; shift
  python bench.py "$@" > $O/$tag.json 2> $O/$tag.err
  python - "$O/$tag.json" "$tag" <<'EOF'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().splitlines()[-1])
    e = d.get("e2e", {})
    print(sys.argv[2], "ms/step %.3f" % d["ms_per_step"], "value %.3g" % d["value"],
          "e2e %.3g" % e.get("value", 0), "same_rounds", e.get("same_rounds"))
except Exception as ex:
    print(sys.argv[2], "FAILED", ex)
EOF
}
run bench_c3 --steps 5 --warmup 3
run bench_c3_arls --sampler arls-lev --steps 5 --warmup 3 --no-cpu-baseline
run bench_c2 --config c2 --steps 5 --warmup 3 --no-cpu-baseline
run bench_reference_c3 --impl reference --steps 3 --warmup 3
for R in 25 50 75; do
  for S in sts arls-lev; do
    run bench_c4_${S}_r$R --config c4 --sampler $S --rank $R --steps 3 --warmup 3
  done
done
