timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_cost5$' -s 1 -c 1 -o gpurun_out/c5prof python tools/run_cost.py --batch 4 --reps 2 > gpurun_out/c5ncu.log 2>&1
ls -la gpurun_out/
