for cfg in C2 C3 C5; do for d in 2 3 4 6 8 16; do echo "$cfg act_div=$d: $(EXACTZ_ACT_DIV=$d python tools/quick_time.py $cfg 2>&1 | grep 'rep 2')"; done; done
