set -x
for v in 1 0; do CD_SYMM_IN_PANEL=$v N=1024 python tools/time_mid.py; CD_SYMM_IN_PANEL=$v N=2048 ONLY=rev python tools/time_mid.py; done
CD_SYMM_IN_PANEL=0 CD_LL_PIECES=16 N=1024 ONLY=rev python tools/time_mid.py
CD_SYMM_IN_PANEL=0 CD_LL_PIECES=4 N=1024 ONLY=rev python tools/time_mid.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_symm_ll -s 100 -c 1 -o gpurun_out/r02_symm_full -f python tools/prof_rev.py --n 16384 > gpurun_out/ncu_symm.log 2>&1
echo ncu rc=$?
