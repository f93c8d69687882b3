for lib in paper_2208_12350_b200/libsw_b200.so build_var/libsw_abl4.so; do SW_B200_LIB=$lib timeout 600 python tools/quick_time.py c5 2>&1 | grep -E "stages|fwd kernel"; done
