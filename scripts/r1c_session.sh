#!/bin/bash
# Round-1 validation pass: every GPU test, every bench config, ncu of the
# config-4 scan. Usage: bash scripts/r1c_session.sh TAG
set -u
TAG=${1:-r1c}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"
for c in 2 1 3 4 5; do
  timeout 1500 python bench.py --config $c > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c rc=$?"
done
[ -n "${SKIP_NCU:-}" ] || bash scripts/ncu_ivf_tc.sh $TAG
