python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 --config c1 > gpurun_out/ref_c1_torchrun.json 2> gpurun_out/ref_c1_torchrun.err
echo done
