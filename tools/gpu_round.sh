#!/bin/bash
# One gpurun call: GPU tests, smoke, bench on every config, the reference arm,
# ncu launch lists and one `ncu --set full` capture per dominant kernel.
# Outputs under gpurun_out/$TAG/ (summarised into profiles/ by tools/ncu_summary.py).
# usage: gpurun -- 'bash tools/gpu_round.sh TAG [parts...]'   parts: tests smoke bench ref dist ncu full
TAG=${1:-r02}
shift
PARTS=${*:-"tests smoke bench ref dist ncu full"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
has() { [[ " $PARTS " == *" $1 "* ]]; }
if has tests; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu.txt
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
  echo "smoke exit $?" >> $OUT/smoke.txt
fi
if has bench; then
  timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
  for C in C1 C3 C4 C4P C5; do
    timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-cpu > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  done
fi
if has ref; then
  timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
fi
if has dist; then  # the N > 1 bench path on ONE GPU: 2 ranks share cuda:0, gloo all-reduce (no kernel waits on another rank)
  IHS_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-cpu > $OUT/bench_2ranks_gloo.json 2> $OUT/bench_2ranks_gloo.err
fi
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-ttt"
if has ncu; then
  for C in C1 C2 C3 C4 C5; do
    $B --config $C > $OUT/plain_$C.log 2>&1 &&
    timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$C.csv $B --config $C > $OUT/ncu_launch_$C.log 2>&1
  done
fi
if has full; then
  B1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-ttt"
  $B1 --config C2 > $OUT/plain1_C2.log 2>&1 &&
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:cs_gather_tma -s 3 -c 1 \
    -o $OUT/full_C2 -f $B1 --config C2 > $OUT/ncu_full_C2.log 2>&1
  $B1 --config C3 > $OUT/plain1_C3.log 2>&1 &&
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"csr_sketch|gram_streamk|ols_large" -s 6 -c 3 \
    -o $OUT/full_C3 -f $B1 --config C3 > $OUT/ncu_full_C3.log 2>&1
  $B1 --config C4 > $OUT/plain1_C4.log 2>&1 &&
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"pg_warp" -s 6 -c 1 \
    -o $OUT/full_C4 -f $B1 --config C4 > $OUT/ncu_full_C4.log 2>&1
  $B1 --config C5 > $OUT/plain1_C5.log 2>&1 &&
  timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"sjlt_onepass|sjlt_lists|grad_dense" -s 3 -c 3 \
    -o $OUT/full_C5 -f $B1 --config C5 > $OUT/ncu_full_C5.log 2>&1
  $B1 --config C1 > $OUT/plain1_C1.log 2>&1 &&
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"small_step" -s 3 -c 1 \
    -o $OUT/full_C1 -f $B1 --config C1 > $OUT/ncu_full_C1.log 2>&1
fi
ls -la $OUT
