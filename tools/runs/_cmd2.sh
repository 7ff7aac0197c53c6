set -u
A="--no-e2e --no-cpu-baseline --steps 20 --warmup 5"
TAG=spc bash tools/ab.sh "$A --estimate sorted" main sp_u8 sp_u16 sp_pf64 sp_u8pf64
TAG=sp10 bash tools/ab.sh "$A --estimate sorted --config 10G" main sp_u8 sp_u16 sp_pf64 sp_u8pf64
TAG=scan bash tools/ab.sh "$A --estimate staged" main scan_nobatch scan_minb4
TAG=scan10 bash tools/ab.sh "$A --config 10G" main scan_nobatch scan_minb4
TAG=auto bash tools/ab.sh "--steps 20 --warmup 5 --no-cpu-baseline" main
