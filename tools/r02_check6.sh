cd $GRAFT_REPO_ROOT
o=gpurun_out/${1:-c7}; mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py -m gpu -q -x -k "dense or hybrid or mixed" > $o/pytest.log 2>&1; tail -2 $o/pytest.log
for c in C3 C4 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/bench_$c.json 2> $o/bench_$c.err; python -c "
import json; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['engine'], d['ms_per_step'], d['roofline']['frac'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"face12" -c 2 --csv --log-file $o/f12.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; grep -o '"gpu__time_duration.sum","ns","[0-9,]*"' $o/f12.csv
