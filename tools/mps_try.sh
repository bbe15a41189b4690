export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo mps started
sleep 1
SEQBAL_BARRIER=device timeout 300 python bench.py --gpus 2 --steps 50 --warmup 3 > gpurun_out/b_c2_g2mps.jsonl 2> gpurun_out/b_c2_g2mps.err
SEQBAL_BARRIER=device timeout 300 python bench.py --gpus 4 --steps 50 --warmup 3 > gpurun_out/b_c2_g4mps.jsonl 2> gpurun_out/b_c2_g4mps.err
SEQBAL_BARRIER=device timeout 300 python bench.py --gpus 8 --steps 50 --warmup 3 > gpurun_out/b_c2_g8mps.jsonl 2> gpurun_out/b_c2_g8mps.err
echo quit | nvidia-cuda-mps-control
tail -c 1500 gpurun_out/b_c2_g2mps.err; cat /tmp/mps_log/control.log | tail -5
