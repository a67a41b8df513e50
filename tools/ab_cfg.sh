# A/B of dev builds on given configs: bash tools/ab_cfg.sh TAG "CFG:lib CFG:lib ..." [NLIM]
TAG=$1; PAIRS=$2; NL=${3:-16777216}
for pr in $PAIRS; do c=${pr%%:*}; v=${pr##*:}
  SST_LIB_PATH=$PWD/paper_2003_07065_b200/libsst_$v.so NLIM=$NL python tools/time_cfg.py $c 5
done > gpurun_out/abc_$TAG.log 2>&1
