for lib in paper_2208_12350_b200/libsw_b200.so build_var/libsw_fb4.so build_var/libsw_pk8.so paper_2208_12350_b200/libsw_b200.so; do
  SW_B200_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['value'], d['stage_ms'])"
done
