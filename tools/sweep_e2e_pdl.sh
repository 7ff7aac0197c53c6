for pdl in 0 2; do for r in 1 2; do VBDR_PDL=$pdl timeout 300 python bench.py --no-cpu-baseline > gpurun_out/e2e_pdl$pdl.$r.json 2>/dev/null; done; done
