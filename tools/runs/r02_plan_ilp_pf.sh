# staged plan (best-fit scheduler) ILP and L2-prefetch distance, caida
A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
TAG=ip bash tools/ab.sh "$A" main ilp2 ilp8 pf2 pf0 main
