python tools/ab.py C3,C2,C5 abvar/v1.so abvar/v1.so:TC_MID_GLOBAL_A=0 abvar/v1.so:TC_FINAL_LD4=0 abvar/v1.so:TC_CO_WARP=0
