for n in 256 512 1024; do N=$n ONLY=rev python tools/time_mid.py; CD_SYMM_IN_PANEL=1 N=$n ONLY=rev python tools/time_mid.py; done
