for v in base t512c4k t128c1k t512c2k t1024c4k; do
  L=tools/variants/$v/libvbdr.so; [ $v = base ] && L=paper_1810_13132_b200/_lib/libvbdr.so
  VBDR_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/sv_caida_$v.json 2>/dev/null
  VBDR_LIB=$L timeout 300 python bench.py --config 10G --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/sv_10G_$v.json 2>/dev/null
done
