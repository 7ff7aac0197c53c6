A="--estimate staged --pipeline off --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
TAG=ilp bash tools/ab.sh "$A" main ilp4 ilp16
