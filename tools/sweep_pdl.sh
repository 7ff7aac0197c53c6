# PDL policy sweep: VBDR_PDL=0 (off), 2 (default: all but the gather estimate), 1 (all)
for pdl in 0 2 1; do
  for rep in 1 2; do
    VBDR_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/pdl_caida_$pdl.$rep.json 2>/dev/null
  done
  VBDR_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline --no-e2e --layout packed > gpurun_out/pdl_caidap_$pdl.json 2>/dev/null
  VBDR_PDL=$pdl timeout 300 python bench.py --config 10G --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pdl_10G_$pdl.json 2>/dev/null
  VBDR_PDL=$pdl timeout 300 python bench.py --config bigwin --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pdl_bigwin_$pdl.json 2>/dev/null
done
