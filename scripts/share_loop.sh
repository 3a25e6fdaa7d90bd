mkdir -p gpurun_out/sl
for cfg in "DC_SPIN_MS=120000"; do
  for i in 1 2 3 4; do
    env $cfg CUDA_DEVICE_MAX_CONNECTIONS=8 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2961$i bench.py --gpus 2 --steps 2 --warmup 3 --layers 2 --batch 1 --share-gpu > /dev/null 2> gpurun_out/sl/err.txt
    echo "$cfg run$i rc=$?" >> gpurun_out/sl/res.txt
    grep -o "DC_E[A-Z]*: [a-z ]*(code 0x[0-9a-f]*)" gpurun_out/sl/err.txt | head -1 >> gpurun_out/sl/res.txt
  done
done
