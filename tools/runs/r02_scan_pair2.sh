A="--estimate staged --no-e2e --no-cpu-baseline --steps 30 --warmup 5"
TAG=c bash tools/ab.sh "$A" main pair2 main pair2
TAG=c10 bash tools/ab.sh "--config 10G --estimate sorted --no-e2e --no-cpu-baseline --steps 10 --warmup 5" main pair2
TAG=warm bash tools/ab.sh "$A --flush-mib 1" main pair2
