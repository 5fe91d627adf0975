#!/bin/bash
# experiment: pair kernel correctness + d12 step times (exp build)
export TNC_LIB=$PWD/tools/_libtnc_exp.so
mkdir -p gpurun_out
[ -n "$SKIPTEST" ] || timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -m gpu -k "f16_split or scaled_precision or engine_sycamore" 2>&1 | tail -15
for cfg in ${CFGS:-"5 3"}; do
  set -- $cfg
  TNC_TG2_RS=$1 TNC_TG2_BS=$2 timeout 180 python tools/net_probe.py --net syc53 --depth 12 --split 6 \
    --cuts 45-49,38-45 --slices 1 --json gpurun_out/exp_pair_$1_$2.json > gpurun_out/exp_pair_$1_$2.log 2>&1
  echo "RS $1 BS $2 rc $?"
  python - <<PY
import json
d=json.load(open("gpurun_out/exp_pair_$1_$2.json"))
s=d["steps"]
print("sum %.1f ms"%(1e3*d["steps_sum_s"]), d["amplitude_partial"], " ".join("%d:%.2f"%(x["step"],x["ms"]) for x in s if x["step"] in (11,12,13,14,17,32,33,35)))
PY
done
python -c "
import json; d=json.load(open('gpurun_out/exp_dbg_0.json')); print('old', d['amplitude_partial'])" 2>/dev/null
