A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
TAG=c bash tools/ab.sh "$A" main nc1 nc2 main
TAG=c10 bash tools/ab.sh "--config 10G --estimate sorted --no-e2e --no-cpu-baseline --steps 10 --warmup 5" main nc1 nc2
