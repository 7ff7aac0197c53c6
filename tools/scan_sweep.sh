VBDR_LIB=tools/variants/sb/libvbdr.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny_every or order_split or caida_full_size" 2>&1 | tail -1
for v in sa sb sc sd se; do
  for c in caida 10G; do
    steps=200; [ "$c" = "10G" ] && steps=20
    VBDR_LIB=tools/variants/$v/libvbdr.so timeout 300 python bench.py --config $c --steps $steps --no-e2e --no-cpu-baseline > gpurun_out/p.json 2>gpurun_out/p.err
    python -c "import json;d=json.loads(open('gpurun_out/p.json').read().strip().splitlines()[-1]);k=d['kernels'];print('$v $c', d['value'], 'step', round(d['ms_per_step']*1e3,1), 'scan', round(k['scan']['ms']*1e3,1))" || tail -3 gpurun_out/p.err
  done
done
