#!/bin/bash
# Same-box A/B of the end-to-end C3 step at N=4 (and N=2): Pipe-SGD vs D-Sync,
# ring CTA budget 64 vs 256, two repetitions (box noise).
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_e2e}
mkdir -p $O
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -m gpu -q -rA > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
fi
for rep in 1 2; do
  for np in ${PS:-4}; do
    for ctas in ${CTAS:-64 256}; do
      for mode in pipe_sgd d_sync; do
        timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
          --master-port 29591 bench.py --gpus $np --ctas $ctas --mode $mode --no-allreduce-sweep \
          > $O/bench_n${np}_${mode}_c${ctas}_r$rep.json 2> $O/bench_n${np}_${mode}_c${ctas}_r$rep.err
      done
    done
  done
done
