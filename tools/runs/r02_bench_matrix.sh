# bench.py option matrix on small configs: every combination must exit 0 with a JSON line
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
fail=0
for cfg in tiny caida_bursty; do
 for lay in fast packed stamps; do
  for est in auto gather sorted staged; do
   for pipe in auto off; do
    timeout 300 $B --config $cfg --layout $lay --estimate $est --pipeline $pipe > /tmp/m.json 2>/tmp/m.err || { echo "FAIL $cfg $lay $est $pipe"; tail -2 /tmp/m.err; fail=1; continue; }
    python -c "import json; d=json.load(open('/tmp/m.json')); assert d['value']>0" || { echo "BADLINE $cfg $lay $est $pipe"; fail=1; }
   done
  done
 done
done
for e in loglog pcsa; do timeout 300 $B --config tiny --layout packed --estimator $e > /tmp/m.json 2>/tmp/m.err || { echo "FAIL estimator $e"; tail -2 /tmp/m.err; fail=1; }; done
timeout 300 $B --config tiny --estimator loglog > /tmp/m.json 2>/tmp/m.err || { echo "FAIL loglog fast"; fail=1; }
timeout 300 $B --config tiny --merge nvls > /tmp/m.json 2>/tmp/m.err || { echo "FAIL nvls"; fail=1; }
timeout 300 python bench.py --impl reference --config tiny --steps 3 --warmup 3 > /tmp/m.json 2>/tmp/m.err || { echo "FAIL ref"; fail=1; }
echo matrix_fail=$fail
