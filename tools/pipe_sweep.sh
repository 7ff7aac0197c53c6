for c in caida 10G; do
  for sm in 0 2; do
    steps=200; [ "$c" = "10G" ] && steps=20
    timeout 300 python bench.py --config $c --steps $steps --no-e2e --no-cpu-baseline --scan-mode $sm > gpurun_out/p.json 2>gpurun_out/p.err
    python -c "import json;d=json.loads(open('gpurun_out/p.json').read().strip().splitlines()[-1]);print('$c scan_mode=$sm', d['value'], 'pipelined', round(d['ms_per_step']*1e3,1), 'serial', round(d['ms_per_step_serial']*1e3,1), 'launches', d['gpu_launches'])" || tail -3 gpurun_out/p.err
  done
done
timeout 300 python -m pytest tests/test_gpu_dist.py -q -x -k bench 2>&1 | tail -1
