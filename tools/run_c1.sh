cd /root/repo
mkdir -p gpurun_out/matrix
Q="--no-cpu-baseline --no-allreduce-sweep"
for n in 1 2 4; do
  for mode in pipe_sgd d_sync; do
    tag=$([ $mode = pipe_sgd ] && echo pipe || echo sync)
    if [ $n -eq 1 ]; then timeout 600 python bench.py --gpus 1 --model c1 --codec none --mode $mode --global-batch 100 --steps 300 --warmup 30 $Q > gpurun_out/matrix/c1_${tag}_n$n.json 2>/dev/null
    else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $n --model c1 --codec none --mode $mode --global-batch 100 --steps 300 --warmup 30 $Q > gpurun_out/matrix/c1_${tag}_n$n.json 2>/dev/null; fi
    echo "c1 $tag n$n $?"
  done
done
