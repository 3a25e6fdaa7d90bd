# N = 2 ranks as two processes time-slicing cuda:0 (bench.py --share-gpu,
# self-launched), repeated: counts stalls (DC_ETIMEOUT with its flag record).
mkdir -p gpurun_out/sl
: > gpurun_out/sl/res.txt
for i in $(seq 1 ${1:-10}); do
  CUDA_DEVICE_MAX_CONNECTIONS=8 timeout 300 python bench.py --gpus 2 --steps 2 --warmup 3 --layers 2 --batch 1 \
      --share-gpu > gpurun_out/sl/out$i.txt 2> gpurun_out/sl/err$i.txt
  echo "run$i rc=$?" >> gpurun_out/sl/res.txt
  grep -o "timed out.*" gpurun_out/sl/err$i.txt | head -2 >> gpurun_out/sl/res.txt
done
