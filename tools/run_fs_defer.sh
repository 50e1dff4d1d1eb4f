# k_fwd_sk deferred fixup against the last-arrival fixup (CD_NO_FS_DEFER), forward at mid N
for n in 1024 2048 4096; do
  N=$n ONLY=fwd python tools/time_mid.py; CD_NO_FS_DEFER=1 N=$n ONLY=fwd python tools/time_mid.py
done
