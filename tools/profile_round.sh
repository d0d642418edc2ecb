#!/bin/bash
# Round profiling recipe (run under gpurun): bench line, reference arm, ncu launch list,
# one `ncu --set full` capture each of the step kernel and the reducer.
#   gpurun -- 'bash tools/profile_round.sh r01'   then   python tools/summarize_ncu.py r01
tag=${1:-r01}
O=gpurun_out
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 3200 --warmup 64 > $O/bench_ref.json 2>&1; echo ref_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 320 --warmup 32 --cpu-seconds 0 --no-bert > $O/ncu_list.out 2>&1; echo list_rc=$?
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
  -f -o $O/prof_bert_attn_$tag python tools/bert_bench.py 32 1 1 8 > $O/ncu_bert_attn.out 2>&1; echo bert_attn_rc=$?
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ln_bwd -c 1 \
  -f -o $O/prof_bert_ln_$tag python tools/bert_bench.py 32 1 1 8 > $O/ncu_bert_ln.out 2>&1; echo bert_ln_rc=$?
# C3 (ResNet-18 per-EST BN step): launch list of one step, ncu of the layer-1 convolution
BT_BENCH_WARMUP=1 BT_BENCH_STEPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 400 \
  --csv --log-file $O/resnet_launches.csv python tools/resnet_bench.py > $O/ncu_resnet_list.out 2>&1; echo resnet_list_rc=$?
# the layer-1 3x3 convolution (first halo-tile launch of the first step: implicit GEMM, resident filter)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_halo -s 0 -c 1 \
  -f -o $O/prof_resnet_conv_$tag python tools/resnet_prof.py 16 32 1 > $O/ncu_resnet_conv.out 2>&1; echo resnet_conv_rc=$?
cat $O/bench.json; tail -3 $O/bench.err
