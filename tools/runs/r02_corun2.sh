# shared-memory carveout of the scan / slide kernels at 100 %: the staged estimate's CTAs can then join SMs running them
cp tools/var_build/capexp/libvbdr.so paper_1810_13132_b200/_lib/libvbdr.so
for C in 0 4; do for M in 2 5; do VBDR_CARVEOUT=100 VBDR_SCAN_BLOCKS_PER_SM=$C python tools/pipe_probe.py --scan-mode $M | sed "s/^/co100 cap=$C /"; done; done
