timeout 300 python tools/diag/time_lowfrac.py
