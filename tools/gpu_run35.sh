# remaining bench configs on the last build
mkdir -p gpurun_out/r02n
O=gpurun_out/r02n
timeout 400 python bench.py --impl reference > $O/bench_c2_ref.jsonl 2> $O/bench_c2_ref.err
timeout 600 python bench.py --config c1 --steps 50 > $O/bench_c1.jsonl 2> $O/bench_c1.err
timeout 600 python bench.py --config c3 --steps 50 > $O/bench_c3.jsonl 2> $O/bench_c3.err
timeout 600 python bench.py --config c3 --topology g8n1 --steps 50 > $O/bench_c3_g8n1.jsonl 2> $O/bench_c3_g8n1.err
timeout 900 python bench.py --config c5 > $O/bench_c5.jsonl 2> $O/bench_c5.err
timeout 300 python tools/bench_uniform.py > $O/bench_uniform.jsonl 2> $O/bench_uniform.err
timeout 600 python bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_c2_2p.jsonl 2> $O/bench_c2_2p.err
python tools/summ.py $O/bench_c1.jsonl $O/bench_c3.jsonl $O/bench_c3_g8n1.jsonl $O/bench_c2_2p.jsonl
