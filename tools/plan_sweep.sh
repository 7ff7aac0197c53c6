for v in cl1 cl2 cl4; do
  VBDR_LIB=tools/variants/$v/libvbdr.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "plan" 2>&1 | tail -1
  VBDR_LIB=tools/variants/$v/libvbdr.so timeout 200 python bench.py --estimate plan --steps 200 --no-e2e --no-cpu-baseline > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "import json;d=json.loads(open('gpurun_out/p.json').read().strip().splitlines()[-1]);k=d['kernels'];print('$v', d['value'], d['ms_per_step'], k['estimate']['ms'])" || tail -3 gpurun_out/p.err
done
