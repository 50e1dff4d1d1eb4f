# panel phases by omission at N=1024 (CD_DEBUG_PANEL_SKIP: results wrong; measurement only)
for m in 0 1 2 4 8 15; do CD_DEBUG_PANEL_SKIP=$m N=${N:-1024} python tools/time_mid.py; done
