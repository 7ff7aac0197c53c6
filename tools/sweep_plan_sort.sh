for v in sort0 sort1 sort2; do
  for rep in 1 2; do
    VBDR_LIB=tools/variants/$v/libvbdr.so timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/sort_$v.$rep.json 2>/dev/null
  done
done
