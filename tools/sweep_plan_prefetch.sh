for v in pf1 pf2 pf3 pf2t; do
  L=tools/variants/$v/libvbdr.so; [ $v = base ] && L=paper_1810_13132_b200/_lib/libvbdr.so
  for rep in 1 2; do
    VBDR_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/pf_$v.$rep.json 2>/dev/null
  done
done
