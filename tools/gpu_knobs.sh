# DAG bench step under the inversion / GEMM knobs (value only)
mkdir -p gpurun_out/knobs
one() { echo -n "$* : " >> gpurun_out/knobs/res.txt; env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step'],4), round(d['phases']['inversion']['ms'],4))" >> gpurun_out/knobs/res.txt; }
one PF_X=0
one PF_NSPLIT32=4
one PF_NSPLIT32=16
one PF_NSPLIT64=2
one PF_NSPLIT64=8
one PF_PERSIST_KMIN=256
one PF_PERSIST_KMIN=1024
one PF_GEMM_PERSIST=0
one PF_TRTRI_SPINE=0
one PF_EARLY_ROOT=0
one PF_INV_RECURSIVE=1
one PF_X=1
echo finished >> gpurun_out/knobs/res.txt
