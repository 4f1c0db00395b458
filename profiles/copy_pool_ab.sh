for i in 1 2; do
 echo pool; python profiles/c1_bench.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['gpu_e2e_ms'], d['gpu_e2e_ms_pinned_inputs'], d.get('bit_exact'))"
 python profiles/fold_bench.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e_ms_by_output_buffers'])"
 echo spawn; IRL_B200_LIB=build/variants/libirl_spawn.so python profiles/c1_bench.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['gpu_e2e_ms'], d['gpu_e2e_ms_pinned_inputs'], d.get('bit_exact'))"
 IRL_B200_LIB=build/variants/libirl_spawn.so python profiles/fold_bench.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e_ms_by_output_buffers'])"
done
