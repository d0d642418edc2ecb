# ncu --set full of one launch of each named C4 kernel (2-layer BertJob, 1 warm-up step, 1 step):
#   bash tools/prof_bert_kernels.sh ln_fwd ln_bwd ...    -> gpurun_out/k_<name>.ncu-rep
mkdir -p gpurun_out
export BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1
for k in "$@"; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o gpurun_out/k_$k python tools/bert_bench.py 32 1 2 8 > gpurun_out/k_$k.out 2>&1
done
ls gpurun_out
