# dev: end-to-end time over EXACTZ_SNAP_DIV (when the result's D2H copy starts), C2
for d in 128 512 1024 4096 16384; do echo "snap_div=$d: $(EXACTZ_SNAP_DIV=$d python tools/e2e_time.py 2>&1 | tail -2 | tr '\n' ' ')"; done
