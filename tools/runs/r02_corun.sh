# scan grid capped so it co-resides with the staged estimate in the pipelined step
cp tools/var_build/capexp/libvbdr.so paper_1810_13132_b200/_lib/libvbdr.so
for C in 0 4 3 2; do for M in 2; do VBDR_SCAN_BLOCKS_PER_SM=$C python tools/pipe_probe.py --scan-mode $M | sed "s/^/cap=$C /"; done; done
VBDR_SCAN_BLOCKS_PER_SM=4 python tools/pipe_probe.py --scan-mode 5 | sed "s/^/cap=4 /"
