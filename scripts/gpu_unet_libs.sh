# U-Net timing over library variants (NAR_B200_LIB): event timing + a per-layer launch list each
# usage: LIBS="base:paper_2407_19097_b200/libnar_b200.so m1:scripts/exp/m1.so" [ENVS="K=V ..."] bash scripts/gpu_unet_libs.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lv in $LIBS; do name=${lv%%:*}; lib=${lv#*:}
  echo "== $name"
  env $ENVS NAR_B200_LIB=$PWD/$lib timeout 120 python scripts/prof_unet.py --frames 6 2>&1 | tail -2
  env $ENVS NAR_B200_LIB=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ul_$name.csv python scripts/prof_unet.py --frames 1 > /dev/null 2>&1
done
