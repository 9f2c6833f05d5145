mkdir -p gpurun_out
timeout 300 python tests/diag/esc_dbg.py > gpurun_out/esc_dbg.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python -c "
import sys; sys.path.insert(0,'.')
import datagen, paper_1505_01998_b200 as kb
ctx=kb.Context(); X=kb.to_device(datagen.config_data('C3'))
ctx.select_bandwidth(kb.LSCV_H, X, max_iter=20)
ctx.select_bandwidth(kb.LSCV_H, X, max_iter=20)
" > gpurun_out/ncu_c3.log 2>&1
cat gpurun_out/esc_dbg.txt
