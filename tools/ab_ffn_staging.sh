set -x
for v in "BT_FFN_NB=2" "BT_FFN_NB=1" "BT_FFN_NB=2" "BT_FFN_NB=1"; do env $v python tools/ffn_epi_bench.py; done > gpurun_out/ab_ffn.log 2>&1
for v in "BT_FFN_NB=2" "BT_FFN_NB=1" "BT_FFN_NB=1 BT_PAIR_S6=1"; do echo "== $v"; env $v python tools/gemm_list.py 2; done > gpurun_out/ab_gemmlist.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_bert.py tests/test_gpu_ffn.py -x -q > gpurun_out/ab_tests.log 2>&1; echo TESTS $?
BT_PAIR_S6=1 timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_bert.py -x -q > gpurun_out/ab_tests_s6.log 2>&1; echo TESTS6 $?
