timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -12 > gpurun_out/r2_gputest3.log; cat gpurun_out/r2_gputest3.log
MOBILE_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-configs --no-cpu-baseline --ep-batch 16 > gpurun_out/r2_bench_ws2.json 2> gpurun_out/r2_bench_ws2.err; tail -3 gpurun_out/r2_bench_ws2.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench_ws2.json')); print(json.dumps(d['ep']))"
for kd in little full; do for ctx in 512 64; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:decode_pass -s 3 -c 1 python scripts/prof_dp2.py c3 $kd $ctx 2 2>&1 | grep -E "dram__|lts__|gpu__time" | sed "s/^/$kd ctx$ctx /"
done; done
