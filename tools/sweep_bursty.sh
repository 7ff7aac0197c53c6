# scan modes on packet trains (caida_bursty) vs i.i.d. caida
for lay in fast packed; do
  for m in 1 2 3 5; do
    timeout 300 python bench.py --config caida_bursty --layout $lay --scan-mode $m --no-cpu-baseline --no-e2e > gpurun_out/bu_${lay}_$m.json 2>/dev/null
  done
done
