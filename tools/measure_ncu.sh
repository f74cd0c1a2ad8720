#!/bin/bash
# Measurement pass part 2 (run under gpurun): ncu --set full captures of one steady-state step's
# K2 launches (INT8 and FP16 4K) and of K1 / K3 / K4, summarised on the box into
# gpurun_out/ncu_R.json (tools/ncu_to_profile.py); only the INT8 K2 report is kept (the rest
# would overflow gpurun's 64 MiB copy-back).
set -u
R=${1:-r02}
mkdir -p gpurun_out
for W in llama8b_int8_4k llama8b_fp16_4k; do
  # two steady-state steps' K2 launches (general / FP16 stream / tcgen05 / combine; the last of each kernel is kept)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_" -s 24 -c 8 \
      -o gpurun_out/${R}_ncu_k2_${W} python bench.py --steps 3 --warmup 4 --no-cpu --no-variants --workload $W > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"k3_manage|k1_confidence|k4_quant" -s 8 -c 3 \
    -o gpurun_out/${R}_ncu_k134 python bench.py --steps 3 --warmup 3 --no-cpu --no-variants > /dev/null 2>&1
python tools/ncu_to_profile.py ${R} gpurun_out gpurun_out > gpurun_out/${R}_ncu_summary.txt 2>&1
rm -f gpurun_out/${R}_ncu_k2_llama8b_fp16_4k.ncu-rep gpurun_out/${R}_ncu_k134.ncu-rep
ls -la gpurun_out | tail -20
