# timing of C2 with different tracking thresholds (dev tool)
for d in ${@:-4 8 16 32}; do echo "ACT_DIV=$d"; EXACTZ_ACT_DIV=$d REPS=3 python tools/quick_time.py C2 2>&1 | grep "rep 2"; done
