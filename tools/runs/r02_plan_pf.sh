# C register ranges x L2 prefetch depth of the plan entries (staged plan), caida
A="--estimate staged --no-e2e --no-cpu-baseline --steps 20 --warmup 5"
VBDR_PLAN_RANGES=4 TAG=r4 bash tools/ab.sh "$A" main pf2 pf4 pf8
VBDR_PLAN_RANGES=2 TAG=r2 bash tools/ab.sh "$A" main pf2 pf4
VBDR_PLAN_RANGES=1 TAG=r1 bash tools/ab.sh "$A" main pf2
