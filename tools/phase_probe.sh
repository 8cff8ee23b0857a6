for f in 0 16 32 64 48 80 96 112; do echo "flags=$f"; SDV_PROBE_FLAGS=$f python tools/group_sweep.py 3 110; done
