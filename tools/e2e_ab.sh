for rc in 1 2 4 8; do
  LORA_HOST_ROW_CHUNKS=$rc timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --e2e-steps 5 > gpurun_out/e2e_rc$rc.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e2e_rc$rc.json').read().strip().splitlines()[-1]); print('rc $rc', d['e2e']['ms_per_step'], d['e2e']['value'])"
done
