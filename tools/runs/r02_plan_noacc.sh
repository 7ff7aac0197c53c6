# staged plan, C register ranges, with and without the accumulation (timing only), caida
A="--estimate staged --pipeline off --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
for C in 4 1; do VBDR_PLAN_RANGES=$C TAG=r$C bash tools/ab.sh "$A" c4 c4noacc; done
