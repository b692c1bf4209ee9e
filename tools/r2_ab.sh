python tools/ab.py C3,C2 abvar/v2.so abvar/v2.so:TC_FINAL_DUAL=0 abvar/v2.so:TC_FINAL_THREADS=1024 abvar/v2.so:TC_FINAL_THREADS=256
