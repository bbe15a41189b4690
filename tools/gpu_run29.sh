# the driver's launch form for N > 1 (torchrun), two ranks on the one GPU: both arms
mkdir -p gpurun_out/r02l
O=gpurun_out/r02l
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > $O/torchrun_ours.jsonl 2> $O/torchrun_ours.err; echo "rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $O/torchrun_ref.jsonl 2> $O/torchrun_ref.err; echo "rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --config c4 --gpus 2 --steps 20 --warmup 3 > $O/torchrun_c4.jsonl 2> $O/torchrun_c4.err; echo "rc=$?"
wc -l $O/*.jsonl; tail -3 $O/*.err
python tools/summ.py $O/torchrun_ours.jsonl
