# A/B of variant libraries (tools/build_variant.sh): gpu_variants.sh CONFIG STEPS NAME[:ENV=VAL[,ENV=VAL]]...
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
cfg=$1; steps=$2; shift 2
for spec in "$@"; do
  v=${spec%%:*}; envs=""
  if [[ "$spec" == *:* ]]; then envs=$(echo "${spec#*:}" | tr ',' ' '); fi
  echo "== $spec"
  env $envs BFM_LIB_OVERRIDE=$GRAFT_REPO_ROOT/paper_1905_12154_b200/variants/libbfm_$v.so timeout 300 python tools/ct_ab.py $cfg $steps
done
