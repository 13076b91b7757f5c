mkdir -p gpurun_out
GTS_BENCH_ONE_DEVICE=1 GTS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --workload tloc --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tloc_n2_g37.json 2> gpurun_out/bench_tloc_n2_g37.err
echo rc=$? > gpurun_out/status_g37.txt
GTS_BENCH_ONE_DEVICE=1 GTS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --workload words --n 200000 --nq 2000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_words_n2_g37.json 2> gpurun_out/bench_words_n2_g37.err
echo rc=$? >> gpurun_out/status_g37.txt
GTS_BENCH_ONE_DEVICE=1 GTS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --impl reference --gpus 2 --workload tloc --steps 3 --warmup 3 > gpurun_out/bench_ref_n2_g37.json 2> gpurun_out/bench_ref_n2_g37.err
echo rc=$? >> gpurun_out/status_g37.txt
echo done >> gpurun_out/status_g37.txt
