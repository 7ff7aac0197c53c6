for pl in 24 25 26 27; do
  for lanes in 4 8; do
    timeout 300 python bench.py --config bigwin --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --est-pass-log2 $pl --est-lanes $lanes > gpurun_out/p.json 2>gpurun_out/p.err
    python -c "import json;d=json.loads(open('gpurun_out/p.json').read().strip().splitlines()[-1]);k=d['kernels'];print('pass_log2=$pl lanes=$lanes est', round(k['estimate']['ms'],2), 'ms')" || tail -2 gpurun_out/p.err
  done
done
