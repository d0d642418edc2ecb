# A/B of the FFN GEMMs' epilogue shape: 16 warps x 1 box x 5 stages (default) / 8 x 1 x 6 / 8 x 2 x 5
for i in 1 2; do for v in "BT_FFN_EW=16" "BT_FFN_EW=81" "BT_FFN_EW=8"; do echo "== $v"; env $v python tools/ffn_epi_bench.py | grep ffn; done; done
