#!/bin/bash
# Round-end evidence pass on one B200: full GPU suite, smoke(), the default
# bench line (C2 + C4/C5 legs + CPU arm), the reference arm, the bench launch
# list and one ncu --set full capture of the C2 kernel (exported for
# tools/ncu_digest.py).
TAG=${1:-e}
O=gpurun_out
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?" >> $O/${TAG}_bench.err
timeout 900 python bench.py --impl reference > $O/${TAG}_refarm.json 2> $O/${TAG}_refarm.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --legs none > $O/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_u8_3d -s 2 -c 1 -o $O/${TAG}_prof \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --legs none > $O/${TAG}_ncu_full.log 2>&1
ncu -i $O/${TAG}_prof.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>/dev/null
ncu -i $O/${TAG}_prof.ncu-rep --page source --csv --print-source sass > $O/${TAG}_sass.csv 2>/dev/null
rm -f $O/${TAG}_prof.ncu-rep
tail -3 $O/${TAG}_pytest.log; cat $O/${TAG}_smoke.log; tail -1 $O/${TAG}_bench.err
