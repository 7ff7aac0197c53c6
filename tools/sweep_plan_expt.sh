for v in x4 x5; do
  VBDR_LIB=tools/variants/$v/libvbdr.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/px_$v.json 2>/dev/null
done
