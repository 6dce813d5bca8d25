#!/usr/bin/env bash
# ncu --set full of each member kernel family + the combine kernel, one
# member per process (tools/time_members.py, 1 step).  Run under gpurun:
#   bash tools/ncu_members.sh <tag>
# -> gpurun_out/ncu_<tag>_<member>.ncu-rep
set -u
tag=${1:-cur}
nb=${NB:-1048576}
out=gpurun_out
mkdir -p $out
cap() {  # name kernel-regex member-spec [batch]
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$2" -c 1 \
    -o $out/ncu_${tag}_$1 -f python tools/time_members.py "$3" --nb $nb --steps 1 \
    --batch ${4:-128} > $out/ncu_${tag}_$1.log 2>&1 || echo "ncu $1 failed"
}
cap mlp256_tmem member_mlp2_tmem mlp:784,256,10
cap mlp512_pair member_mlp2_pair mlp:784,512,10
cap cnn_conv conv_stack cnn
cap cnn_head member_mlp2 cnn
cap mlp1024_pair member_mlp2_pair mlp:784,1024,10
cap mlp512x2_dense dense_pair mlp:784,512,512,10
cap combine combine_kernel mlp:784,128,10
