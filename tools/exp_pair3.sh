#!/bin/bash
export TNC_LIB=$PWD/tools/_libtnc_exp.so
for lu in ${LEADS:-1:16 2:16 2:8 4:8 1:64}; do lead=${lu%:*}; export TNC_TG2_UNIT=${lu#*:}; echo -n "unit $TNC_TG2_UNIT ";
  TNC_TG2_LEAD=$lead timeout 50 python tools/net_probe.py --net syc53 --depth 12 --split 6 \
    --cuts 45-49,38-45 --slices 1 --json gpurun_out/exp_p3_$lead.json > gpurun_out/exp_p3_$lead.log 2>&1
  echo -n "lead $lead rc $? "
  python - <<PY
import json
d=json.load(open("gpurun_out/exp_p3_$lead.json"))
s=d["steps"]
print("sum %.1f ms"%(1e3*d["steps_sum_s"]), d["amplitude_partial"], " ".join("%d:%.2f"%(x["step"],x["ms"]) for x in s if x["step"] in (11,12,13,14,17,32,33,35)))
PY
done
