# k_symm_ll deferred fixup (CD_NO_LL_DEFER restores the last-arrival fixup) and the in-panel SYMM
# (CD_SYMM_IN_PANEL=0: every trailing update on k_symm_ll), reverse at mid N
for n in 1024 2048 4096 8192; do
  N=$n ONLY=rev python tools/time_mid.py
  CD_SYMM_IN_PANEL=0 N=$n ONLY=rev python tools/time_mid.py
  CD_NO_LL_DEFER=1 N=$n ONLY=rev python tools/time_mid.py
done
