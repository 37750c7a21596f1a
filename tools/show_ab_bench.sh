#!/bin/bash
for f in gpurun_out/ab_$1_*.log; do printf "%s %s %s %s\n" "$f" "$(tail -1 $f)" "$(grep -o '"ms_per_step": [0-9.]*' $f)" "$(grep -o '"sm_mhz": [0-9.]*' $f)"; done
