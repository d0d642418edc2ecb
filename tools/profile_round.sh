#!/bin/bash
# Round profiling recipe (run under gpurun): bench line, reference arm, ncu launch list,
# one `ncu --set full` capture each of the step kernel and the reducer.
#   gpurun -- 'bash tools/profile_round.sh r02'   then copy gpurun_out/prof_out/* into profiles/
tag=${1:-r02}
O=gpurun_out
mkdir -p $O
python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo pytest_rc=$?
# the driver's command first (the headline), then the long default run
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2>&1; echo ref_rc=$?
python bench.py --no-bert > $O/bench_long.json 2> $O/bench_long.err; echo bench_long_rc=$?
python bench.py --gpus 2 --steps 100 --warmup 5 --no-bert --no-reducer --cpu-seconds 0 > $O/bench_n2.json 2> $O/bench_n2.err; echo n2_rc=$?
python tools/xdev_timing.py > $O/xdev_timing.json 2>&1; python tools/xdev_stages.py 2 4 8 > $O/xdev_stages.txt 2>&1
python tools/stage_cycles.py 8,4,20 8,4,100 > $O/stage_cycles.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv \
  python bench.py --steps 20 --warmup 5 --cpu-seconds 0 --no-bert --no-reducer > $O/ncu_list.out 2>&1; echo list_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_step -s 3 -c 1 -f -o $O/prof_mlp_$tag \
  python bench.py --steps 64 --warmup 32 --cpu-seconds 0 --no-reducer --no-bert > $O/ncu_mlp.out 2>&1; echo mlp_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reduce_fast -s 2 -c 1 -f -o $O/prof_reduce_$tag \
  python bench.py --steps 64 --warmup 32 --cpu-seconds 0 --no-bert > $O/ncu_red.out 2>&1; echo red_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -f -o $O/prof_gemm_$tag \
  python tools/gemm_bench.py 8192,8192,8192 > $O/ncu_gemm.out 2>&1; echo gemm_rc=$?
# C4 (BERT-base per-EST step): launch list of one step (1 warm-up + 1 step), ncu of the FFN forward
# GEMM (3rd GEMM launch of a step: T x 3072 x 768, bias+GELU epilogue), attention backward, LN backward
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 360 -c 400 \
  --csv --log-file $O/bert_launches.csv python tools/bert_bench.py 32 1 12 8 > $O/ncu_bert_list.out 2>&1; echo bert_list_rc=$?
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 \
  -f -o $O/prof_bert_gemm_$tag python tools/bert_bench.py 32 1 1 8 > $O/ncu_bert_gemm.out 2>&1; echo bert_gemm_rc=$?
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -c 1 \
  -s 2 -f -o $O/prof_bert_attn_$tag python tools/bert_bench.py 32 1 2 8 > $O/ncu_bert_attn.out 2>&1; echo bert_attn_rc=$?
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ln_bwd -s 2 -c 1 \
  -f -o $O/prof_bert_ln_$tag python tools/bert_bench.py 32 1 2 8 > $O/ncu_bert_ln.out 2>&1; echo bert_ln_rc=$?
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ln_fwd -s 2 -c 1 \
  -f -o $O/prof_bert_lnf_$tag python tools/bert_bench.py 32 1 2 8 > $O/ncu_bert_lnf.out 2>&1; echo bert_lnf_rc=$?
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 \
  -f -o $O/prof_bert_attnf_$tag python tools/bert_bench.py 32 1 2 8 > $O/ncu_bert_attnf.out 2>&1; echo bert_attnf_rc=$?
# C3 BatchNorm kernels (statistics pass, apply, backward: the 3rd launch of each)
for k in stats_kernel bn_apply_kernel bn_bwd_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o $O/prof_resnet_${k}_$tag \
    python tools/resnet_prof.py 16 32 1 > $O/ncu_resnet_$k.out 2>&1; echo resnet_${k}_rc=$?
done
python tools/resnet_prof.py 16 32 1 > $O/resnet_prof.txt 2>&1
python tools/bert_prof.py 32 12 8 > $O/bert_prof.txt 2>&1; python tools/gemm_list.py 2 > $O/gemm_list.txt 2>&1
# C3 (ResNet-18 per-EST BN step): launch list of one step, ncu of the layer-1 convolution
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 400 \
  --csv --log-file $O/resnet_launches.csv python tools/resnet_bench.py > $O/ncu_resnet_list.out 2>&1; echo resnet_list_rc=$?
# the layer-1 3x3 convolution (first halo-tile launch of the first step: implicit GEMM, resident filter)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_halo -s 0 -c 1 \
  -f -o $O/prof_resnet_conv_$tag python tools/resnet_prof.py 16 32 1 > $O/ncu_resnet_conv.out 2>&1; echo resnet_conv_rc=$?
# summaries on the box (the .ncu-rep files are too large to bring back): profiles-format text + traffic.json
BT_PROF_OUT=$O/prof_out python tools/summarize_ncu.py $tag > $O/summarize.out 2>&1; echo summarize_rc=$?
rm -f $O/*.ncu-rep
cat $O/bench.json; tail -3 $O/bench.err
