# round-2 final measurement pass (one B200): GPU suite, every bench line, reference arm,
# launch list, one ncu --set full capture of the caida step's kernels per layout
set -u
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_caida_fast.json 2> gpurun_out/bench_caida_fast.err; echo bench=$?
timeout 300 python bench.py --layout packed --no-cpu-baseline > gpurun_out/bench_caida_packed.json 2> gpurun_out/bench_caida_packed.err; echo packed=$?
timeout 300 python bench.py --layout stamps --no-cpu-baseline > gpurun_out/bench_caida_stamps.json 2> gpurun_out/bench_caida_stamps.err; echo stamps=$?
timeout 600 python bench.py --config 10G --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_10G_fast.json 2> gpurun_out/bench_10G.err; echo b10G=$?
timeout 600 python bench.py --config 10G --layout stamps --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bench_10G_stamps.json 2> gpurun_out/bench_10G_stamps.err; echo b10Gs=$?
timeout 900 python bench.py --config bigwin --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bigwin_fast.json 2> gpurun_out/bench_bigwin.err; echo bigwin=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref=$?
A="--steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/ncu_launches.log 2>&1; echo ncu_l=$?
for L in fast packed; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_slide|k_estimate" -s 9 -c 3 -o gpurun_out/prof_final_$L python bench.py $A --estimate staged --pipeline off --layout $L > gpurun_out/ncu_full_$L.log 2>&1; echo ncu_$L=$?
done
