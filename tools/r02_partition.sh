#!/bin/bash
# Green-context comm partition adopted as the engine policy: focused tests + N=4 / N=1 benches.
cd "$(dirname "$0")/.."
O=gpurun_out/${TAG:-r02_partition}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -k "partition or overlaps" > $O/pytest.log 2>&1
echo "pytest exit $?" >> $O/pytest.log
run4() {  # name steps args...
  local name=$1 steps=$2; shift 2
  timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29733 bench.py --gpus 4 --no-allreduce-sweep --steps $steps "$@" > $O/$name.json 2> $O/$name.err
}
run4 c3_pipe 20 --model c3
run4 c3_dsync 20 --model c3 --mode d_sync
run4 c2_pipe 60 --model c2
run4 c2_pipe_sms32 60 --model c2 --comm-sms 32 --ctas 128
run4 c1_pipe 200 --model c1
timeout 300 python bench.py --no-allreduce-sweep --no-cpu-baseline > $O/n1_c3.json 2> $O/n1_c3.err
timeout 300 python bench.py --no-allreduce-sweep --no-cpu-baseline --comm-sms 48 --ctas 192 > $O/n1_c3_sms48.json 2> $O/n1_c3_sms48.err
