#!/bin/bash
# k_step_sw vs the layer-split k_step_sw4 at config 2: per-launch cost fit (tools/advance_cost.py)
for nlw in 0 1 2 3; do
  echo "nlw=$nlw $(SFW_SW_NLW=$nlw SFW_STEP_VERBOSE=1 python tools/advance_cost.py 2>&1 | grep -E '^\{|k_step_sw' | tr '\n' ' ')"
done
