# final build: multi-GPU suite (incl. full size) + bench lines at 2 and 4 GPUs
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r02_multi4_final3.log 2>&1; echo multi rc=$?; tail -1 gpurun_out/r02_multi4_final3.log
run() { n=$1; shift; tag=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@" > gpurun_out/r02_final3_n${n}_$tag.log 2>&1; echo "n=$n $tag rc=$?"; tail -1 gpurun_out/r02_final3_n${n}_$tag.log | cut -c1-200; }
run 2 fine384 --workload fine384_odf64 --steps 100 --warmup 10 --no-e2e
run 4 fine384 --workload fine384_odf64 --steps 100 --warmup 10 --no-e2e
run 2 fine768 --workload fine768_odf64 --steps 100 --warmup 10 --no-e2e
run 4 fine768 --workload fine768_odf64 --steps 100 --warmup 10 --no-e2e
run 2 small192 --workload small192_odf1 --steps 200 --warmup 10 --no-e2e
run 4 small192 --workload small192_odf1 --steps 200 --warmup 10 --no-e2e
run 2 weak1536_20 --steps 20 --warmup 5
run 4 weak1536_20 --steps 20 --warmup 5
