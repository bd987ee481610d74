# N > 1 plumbing of bench.py on a one-GPU box: 2 ranks on GPU 0 over gloo (timings contended; checks the
# sharding, max-over-ranks timing and the JSON line), then the reference arm under torchrun
O=gpurun_out/plumb
mkdir -p $O
for c in c4 c2; do
  NTT_BENCH_PLUMBING_1GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config $c --steps 3 --warmup 3 \
    > $O/n2_$c.json 2> $O/n2_$c.err; echo "n2 $c rc=$? $(tail -c 400 $O/n2_$c.json)"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > $O/ref_n2.json 2> $O/ref_n2.err; echo "ref n2 rc=$? $(tail -c 300 $O/ref_n2.json)"
timeout 300 python bench.py --gpus 2 --steps 2 > $O/selflaunch.json 2> $O/selflaunch.err; echo "self-launch on 1 GPU rc=$? $(tail -c 200 $O/selflaunch.err)"
