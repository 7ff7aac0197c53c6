for c in caida caida_bursty; do for lay in fast packed; do
  timeout 300 python bench.py --config $c --layout $lay --no-cpu-baseline --no-e2e > gpurun_out/dd_${c}_$lay.json 2>/dev/null
done; done
