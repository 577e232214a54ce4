#!/bin/bash
O=gpurun_out/r2o
mkdir -p $O
timeout 600 python bench.py --force-sharded --steps 10 --warmup 3 --e2e-steps 2 > $O/fs.json 2>$O/fs.err; echo rc=$?
python -c "import json;d=json.load(open('$O/fs.json'));print(d['ms_per_step'], d['gather_to_rank0_ms'], d['result_check'])"
timeout 600 python tools/dist_pull_bench.py 8 28
timeout 600 python tools/dist_pull_bench.py 2 28
timeout 600 python -m pytest tests/test_shard_gpu.py -x -q -k "device_counts or dist_build" 2>&1 | tail -2
