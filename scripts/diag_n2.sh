O=gpurun_out/diag; mkdir -p $O
run() { local tag=$1; shift; timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu-baseline "$@" > $O/$tag.json 2> $O/$tag.err; echo "$tag rc=$? $(tail -c 300 $O/$tag.json | grep -o '"value": [0-9.]*' | head -1)"; }
run mix_eager --eager
DM_NCCL_ONE_PG=1 run mix_graph_onepg
run mix_graph
