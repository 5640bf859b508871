#!/bin/bash
# One gpurun call: GPU tests, smoke, bench on every config, the reference arm,
# ncu launch lists and one `ncu --set full` capture per dominant kernel.
# Outputs under gpurun_out/$TAG/ (summarised into profiles/ by tools/ncu_summary.py).
# usage: gpurun -- 'bash tools/gpu_round.sh TAG [parts...]'   parts: probe tests smoke bench dist ncu
TAG=${1:-r01}
shift
PARTS=${*:-"tests smoke bench dist ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
has() { [[ " $PARTS " == *" $1 "* ]]; }
if has probe; then
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/probe tools/probe/probe.cu > $OUT/probe_build.txt 2>&1 &&
    timeout 300 /tmp/probe > $OUT/probe.txt 2>&1
fi
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu.txt
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
  echo "smoke exit $?" >> $OUT/smoke.txt
fi
if has bench; then
  timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
  for C in C1 C3 C4 C4P C5; do
    timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  done
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
fi
if has dist; then  # the N > 1 bench path on ONE GPU: 2 ranks share cuda:0, gloo all-reduce (no kernel waits on another rank)
  IHS_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-cpu > $OUT/bench_2ranks_gloo.json 2> $OUT/bench_2ranks_gloo.err
fi
if has ncu; then
  NCU=/usr/local/cuda/bin/ncu
  for C in C2 C3 C4 C5; do
    python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu --no-ttt > $OUT/plain_$C.log 2>&1 &&
    timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$C.csv python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu --no-ttt \
      > $OUT/ncu_launch_$C.log 2>&1
  done
  B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-ttt"
  $B --config C2 > $OUT/plain1_C2.log 2>&1 &&
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:cs_gather_tma -s 3 -c 1 \
    -o $OUT/full_C2 -f $B --config C2 > $OUT/ncu_full_C2.log 2>&1
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"gram_ols|reduce_rows_last" -s 6 -c 2 \
    -o $OUT/full_C2_factor -f $B --config C2 > $OUT/ncu_full_C2_factor.log 2>&1
  $B --config C3 > $OUT/plain1_C3.log 2>&1 &&
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"gram_streamk|csr_sketch|ols_cg" -s 9 -c 3 \
    -o $OUT/full_C3 -f $B --config C3 > $OUT/ncu_full_C3.log 2>&1
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:csr_sketch -s 3 -c 1 \
    -o $OUT/full_C3_csr -f $B --config C3 > $OUT/ncu_full_C3_csr.log 2>&1
  $B --config C4 > $OUT/plain1_C4.log 2>&1 &&
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"pg_warp|cs_gather_tma" -s 6 -c 2 \
    -o $OUT/full_C4 -f $B --config C4 > $OUT/ncu_full_C4.log 2>&1
  $B --config C5 > $OUT/plain1_C5.log 2>&1 &&
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:cs_gather_tma -s 6 -c 1 \
    -o $OUT/full_C5 -f $B --config C5 > $OUT/ncu_full_C5.log 2>&1
fi
ls -la $OUT
