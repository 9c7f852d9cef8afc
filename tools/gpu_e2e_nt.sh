# e2e (cfg2, 32 slices per call) vs packer store kind and pipeline chunk size, alternating
for r in 1 2; do
  for cfg in "1 2097152" "0 2097152" "0 1048576" "0 524288" "1 1048576"; do
    set -- $cfg
    VKM_PACK_NT=$1 VKM_CHUNK_EVENTS=$2 timeout 300 python tools/trace_batch.py 2>&1 | tail -1 | sed "s/^/nt=$1 chunk=$2 /"
  done
done
