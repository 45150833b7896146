#!/bin/bash
# Final-build evidence: the config-2 step's launch list (ncu, after the same command exited 0 without
# it) and one --set full capture of an 8-wave int8 launch.
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sub"
timeout 600 $CMD > gpurun_out/fn_pre.json 2> gpurun_out/fn_pre.err; echo plain_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/fn_pre.json')); r=d['roofline']; print('ms_per_step', d['ms_per_step'], 'int8', r['kernel_ms'], 'create', r['create_ms'], 'share', r['kernel_ms']/d['ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/fn_launches.csv $CMD > /dev/null 2>&1; echo ncu_launch_rc=$?
python tools/launch_summary.py gpurun_out/fn_launches.csv | head -16
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ozaki_trsm -s 16 -c 1 -o gpurun_out/fn_hot python bench.py --m 833536 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sub > gpurun_out/fn_ncu.log 2>&1; echo ncu_full_rc=$?
ncu -i gpurun_out/fn_hot.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','sm__cycles_elapsed.avg.per_second','launch__grid_size','l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed']
for w in want:
  for i,k in enumerate(h):
    if k==w: print(w, rows[1][i], v[i])
"
