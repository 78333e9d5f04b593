# compute-sanitizer memcheck + racecheck over every kernel instantiation / lowering path:
# common kernel (swap-AB ragged pieces, MN-major B), on-chip cluster split-K (s=2 and s=4),
# global-workspace split-K, eight-warp epilogue (natural BMM table and forced Dense), CTA-pair kernel;
# round 2: TMA tail stores, bulk row stores, overflow split, 32-column pieces with param-space descriptors.
export PYTHONUNBUFFERED=1
OUT=${OUT:-gpurun_out/sanitize.txt}
: > $OUT
run() {  # label, env..., script
  local label=$1; shift
  for tool in memcheck racecheck; do
    extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
    echo "== $tool: $label" >> $OUT
    timeout 300 env "$@" compute-sanitizer --tool $tool $extra python ${SCRIPT} 2>&1 \
      | grep -E "rel err|ERROR SUMMARY|RACECHECK SUMMARY|Error|error" | grep -v "^\[\[" | head -8 >> $OUT
  done
}
SCRIPT=scripts/one_dense.py run "swap-AB ragged j pieces" M=130 N=1000 K=256 ORIENT=1
SCRIPT=scripts/one_dense.py run "B [K,N] MN-major" M=64 N=300 K=100 ORIENT=0 LAYOUT=kn
SCRIPT=scripts/one_dense.py run "on-chip cluster split-K s=2" M=300 N=768 K=1024 ORIENT=-1
SCRIPT=scripts/one_dense.py run "on-chip cluster split-K s=4" M=128 N=768 K=4096 ORIENT=-1
SCRIPT=scripts/one_dense.py run "global-workspace split-K" FTB_SPLIT_CLUSTER=0 M=300 N=768 K=1024 ORIENT=-1
SCRIPT=scripts/one_dense.py run "eight-warp epilogue (forced), Dense" FTB_EPI8=1 M=1000 N=2304 K=512 ORIENT=-1
SCRIPT=scripts/one_bmm.py run "eight-warp epilogue (natural), BMM 192x64x64x64" B=192 M=64 N=64 K=64
SCRIPT=scripts/one_dense.py run "large Dense (CTA-pair candidate)" M=2048 N=3072 K=768 ORIENT=-1
SCRIPT=scripts/one_bmm.py run "TMA tail stores, scores T=95 (padded rows)" B=384 M=95 N=95 K=64 LAYOUT=nk
SCRIPT=scripts/one_bmm.py run "bulk row stores, scores T=95 (compact rows)" COMPACT=1 B=64 M=95 N=95 K=64 LAYOUT=nk
SCRIPT=scripts/one_dense.py run "overflow split (153 items)" M=2144 N=2304 K=768 ORIENT=-1
SCRIPT=scripts/one_dense.py run "32-column pieces, param-space TMA descriptors" M=160 N=768 K=768 ORIENT=-1
cat $OUT
