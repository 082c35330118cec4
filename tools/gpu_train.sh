mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -k "world2 or train or determinism" > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests.log
for ov in 0 1; do
FS4D_OVERLAP_ALLREDUCE=$ov timeout 600 python bench.py --workload train --steps 10 --warmup 3 --no-cpu > gpurun_out/train_ov$ov.json 2> gpurun_out/train_ov$ov.err; echo train$ov=$?
python -c "import json;d=json.loads(open('gpurun_out/train_ov$ov.json').read().strip().splitlines()[-1]);print('ov$ov', d['value'], d['ms_per_step'])"
done
