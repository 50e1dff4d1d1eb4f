#!/bin/bash
# Measurement: cooperative panel grid cap (CD_PANEL_GRID) against the default (every co-resident CTA)
# at mid N, reverse and forward (tools/time_mid.py, L2 flushed between calls).
for n in ${NS:-1024 2048 4096}; do
  for g in ${GRIDS:-0 112 74 48 32}; do
    echo "grid=$g"; CD_PANEL_GRID=$g N=$n python tools/time_mid.py
  done
done
