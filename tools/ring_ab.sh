# pageable staging variants: piece size (MiB) x streaming / cached stores; pinned as the reference
python tools/pcie_diag.py C3 2>&1 | head -2
for v in "TC_RING_CHUNK_MB=16 TC_COPY_NT=1" "TC_RING_CHUNK_MB=8 TC_COPY_NT=0" "TC_RING_CHUNK_MB=4 TC_COPY_NT=0" "TC_RING_CHUNK_MB=16 TC_COPY_NT=1" "TC_RING_CHUNK_MB=8 TC_COPY_NT=0"; do
  echo "== $v"; env $v python tools/e2e_steps.py C3 10 2>&1 | tail -2 | cut -c1-120
done
