# ncu --set full of the C3 BatchNorm kernels (statistics pass, apply, backward): the 3rd launch of each
mkdir -p gpurun_out
for k in stats_kernel bn_apply_kernel bn_bwd_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -f -o gpurun_out/k_$k python tools/resnet_prof.py 16 32 1 > gpurun_out/k_$k.out 2>&1
done
python tools/resnet_prof.py 16 32 1 > gpurun_out/resnet_prof.txt 2>&1
