#!/bin/bash
# One measurement pass for the round (run under gpurun). Outputs land in gpurun_out/.
#   gpurun --timeout 2400 -- 'bash tools/measure_round.sh r01'
set -u
R=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${R}_gpu.csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${R}_pytest_gpu.txt 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${R}_bench_int8.json 2> gpurun_out/${R}_bench_int8.err
for W in llama8b_int8_4k_decode llama8b_fp16_4k llama8b_int8_4k_model llama8b_niah_32k qwen32b_pyramid; do
  timeout 600 python bench.py --steps 50 --warmup 5 --workload $W --no-cpu > gpurun_out/${R}_bench_$W.json 2> gpurun_out/${R}_bench_$W.err
done
timeout 600 python bench.py --steps 50 --warmup 5 --workload gpt2_fp16 > gpurun_out/${R}_bench_gpt2.json 2> gpurun_out/${R}_bench_gpt2.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_bench_reference.err
bash tools/sweep.sh ${R}
for W in llama8b_int8_4k llama8b_fp16_4k; do
  # launch list: prefill, 3 warm-up and 2 timed steps (+ the e2e leg); per-kernel means are taken
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${R}_launches_${W}.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu --workload $W > /dev/null 2>&1
  # two steady-state steps' K2 launches (general / FP16 stream / tcgen05 / combine; the last of each kernel is kept)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_" -s 24 -c 8 \
      -o gpurun_out/${R}_ncu_k2_${W} python bench.py --steps 3 --warmup 4 --no-cpu --workload $W > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"k3_manage|k1_confidence|k4_quant" -s 8 -c 3 \
    -o gpurun_out/${R}_ncu_k134 python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out | tail -40
