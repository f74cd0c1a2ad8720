#!/bin/bash
# One measurement pass for the round, part 1 (run under gpurun): GPU tests, every bench line,
# the reference arm, the C5 batch sweep and the ncu launch lists. Outputs land in gpurun_out/.
#   gpurun --timeout 2400 -- 'bash tools/measure_round.sh r02'   (then tools/measure_ncu.sh r02)
set -u
R=${1:-r02}
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
for W in llama8b_int8_4k llama8b_fp16_4k gpt2_fp16; do
  # launch list: prefill, warm-up and 2 timed steps (+ the e2e leg); per-kernel means are taken
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${R}_launches_${W}.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu --no-variants --workload $W > /dev/null 2>&1
done
ls -la gpurun_out | tail -40
