for m in 5 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --scan-mode $m > gpurun_out/pipe_serial_$m.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --scan-mode $m --pipeline > gpurun_out/pipe_pipe_$m.json 2>/dev/null
done
