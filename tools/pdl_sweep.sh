timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or plan or loopback or sweep" 2>&1 | tail -1
for rep in 1 2; do
for v in pdl0 pdl1; do
  for c in caida 10G; do
    steps=200; [ "$c" = "10G" ] && steps=20
    VBDR_LIB=tools/variants/$v/libvbdr.so timeout 300 python bench.py --config $c --steps $steps --no-e2e --no-cpu-baseline > gpurun_out/p.json 2>gpurun_out/p.err
    python -c "import json;d=json.loads(open('gpurun_out/p.json').read().strip().splitlines()[-1]);k=d['kernels'];print('$v $c', d['value'], 'step', round(d['ms_per_step']*1e3,1), 'sum', round(sum(k[x]['ms'] for x in ['scan','merge','slide','estimate'])*1e3,1), 'slide', round(k['slide']['ms']*1e3,1))" || tail -3 gpurun_out/p.err
  done
done
done
