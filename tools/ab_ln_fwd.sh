# LN forward with parameters through the read-only L1 path (4 blocks / SM): tests + timing + ncu
timeout 900 python -m pytest tests/test_gpu_bert.py tests/test_gpu_bert_peer.py -x -q > gpurun_out/ln_tests.log 2>&1; echo TESTS $?
tail -2 gpurun_out/ln_tests.log
python tools/bert_prof.py 32 12 8 > gpurun_out/ln_bert_prof.txt 2>&1; grep -i "ln_fwd\|ln_bwd\|total\|ms" gpurun_out/ln_bert_prof.txt | head -20
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ln_fwd -s 2 -c 1 \
  -f -o gpurun_out/prof_bert_lnf_r02 python tools/bert_bench.py 32 1 2 8 > gpurun_out/ncu_bert_lnf.out 2>&1; echo lnf_rc=$?
ncu -i gpurun_out/prof_bert_lnf_r02.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__warps_active.avg.pct_of_peak_sustained_active','launch__occupancy_limit_shared_mem','launch__registers_per_thread','launch__grid_size']:
    if k in h: print(k, v[h.index(k)])
"
rm -f gpurun_out/*.ncu-rep
