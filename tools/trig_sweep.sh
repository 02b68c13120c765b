#!/bin/bash
# early-trigger (griddepcontrol.launch_dependents) sweep: rebuild per WK_TRIG_MASK, bench each
for mask in ${MASKS:-0 1 2 4 8}; do
  WK_EXTRA_NVCC_FLAGS="-DWK_TRIG_MASK=$mask" python -c "from paper_2505_02922_b200 import _build; _build.build(force=True)" || continue
  echo "mask=$mask $(bash tools/ab_env.sh WK_PDL 1)"
done
