# staging-ring parameters of the host entries (capi.cu / hostpool.cpp) on the box
for mb in ${MBS:-4 8 16}; do for th in ${THS:-16}; do for g in ${GRAINS:-32768}; do
  echo "== mb=$mb threads=$th grain=$g"; SDFGB_STAGE_MB=$mb SDFGB_HOST_THREADS=$th SDFGB_HOST_GRAIN=$g python tools/e2e_probe.py ${MOTIFS:-query histogram} 2>&1 | grep -v "host threads"
done; done; done
