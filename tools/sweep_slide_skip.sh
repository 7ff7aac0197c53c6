for rep in 1 2; do
  VBDR_LIB=tools/variants/sk1/libvbdr.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/sk1.$rep.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/sk2.$rep.json 2>/dev/null
done
