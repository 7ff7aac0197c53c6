# scan modes at caida (both layouts) and 10G; bench scan times
for cfg in caida 10G; do
  for lay in fast packed; do
    [ $cfg = 10G ] && [ $lay = packed ] && continue
    for m in 1 2 3 4 5 6; do
      [ $lay = packed ] && [ $m = 6 ] && continue
      ST=100; [ $cfg = 10G ] && ST=20
      timeout 300 python bench.py --config $cfg --layout $lay --scan-mode $m --steps $ST --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/sm_${cfg}_${lay}_$m.json 2>/dev/null
    done
  done
done
