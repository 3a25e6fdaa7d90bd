# Re-measure the non-default bench lines at the current defaults (one JSON line each, gpurun_out/lines_rs1/)
mkdir -p gpurun_out/lines_rs1
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" 2> gpurun_out/lines_rs1/$name.err | tail -1 > gpurun_out/lines_rs1/$name.json; }
run mix_b1 --model mixtral-8x7b --batch 1
run mix_b2 --model mixtral-8x7b
run mix_b4 --model mixtral-8x7b --batch 4
run llama_micro4 --micro 4
run llama_ckpt --checkpoint
run llama70b_L8 --model llama3-70b
run off70 --model llama3-70b --layers 16 --batch 1 --offload
