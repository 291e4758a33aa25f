#!/bin/bash
# round 2: 512-thread warp-specialised M2L with staged LF operators (A/B per-level trace), correctness subset,
# the bench through the library's NCCL data plane on one rank, config 5 bench, launch list
mkdir -p gpurun_out
for v in "FDA_GT_WS512=0" "FDA_GT_WS512=1"; do
  echo "== $v" >> gpurun_out/trace_ws512.log
  env $v FDA_TRACE=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/tr.tmp
  grep "fda trace" gpurun_out/tr.tmp | tail -28 >> gpurun_out/trace_ws512.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_devplan.py "tests/test_gpu_configs.py::test_full_oracle_hf_configs" -q -x -s -p no:cacheprovider > gpurun_out/pytest_ws512.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ws512.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --dist --config 3 --steps 5 --warmup 3 > gpurun_out/bench_dist_c3.json 2> gpurun_out/bench_dist_c3.err; echo "exit $?" >> gpurun_out/bench_dist_c3.err
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --verbose > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "exit $?" >> gpurun_out/bench_c5.err
CMD5="python bench.py --config 5 --steps 1 --warmup 3 --no-check"
timeout 900 $CMD5 > gpurun_out/plain_c5.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(gtrans|p2p|csr|s2m|l2t|permute|unpermute|xpack|xunpack)" -c 160 --csv --log-file gpurun_out/launches_c5.csv $CMD5 > gpurun_out/ncu_launch.log 2>&1
echo "launch exit $?" >> gpurun_out/ncu_launch.log
for v in "FDA_M2L_MODE=owned FDA_GT_SLABS=1184" "FDA_M2L_MODE=owned FDA_GT_SLABS=2368" "FDA_M2L_MODE=owned FDA_GT_SLABS=4736"; do
  echo "== $v" >> gpurun_out/trace_ownws.log
  env $v FDA_TRACE=1 timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-check > /dev/null 2> gpurun_out/tr.tmp
  grep "fda trace" gpurun_out/tr.tmp | tail -28 >> gpurun_out/trace_ownws.log
done
FDA_M2L_MODE=owned FDA_GT_SLABS=2368 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_ownws.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ownws.log
