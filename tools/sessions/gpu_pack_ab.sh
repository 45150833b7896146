#!/bin/bash
# oz_pack_kernel through shared memory: shared-state digests vs the previous build (must be equal) and
# the kernel's time (ncu, one create each).
python tools/create_digest.py 1500 4097 10000 > gpurun_out/pk_new.txt 2>&1; echo new_rc=$?
cp paper_1210_7325_b200/libgls.so /tmp/libgls_new.so
cp tools/ab_libs/libgls_base.so paper_1210_7325_b200/libgls.so
python tools/create_digest.py 1500 4097 10000 > gpurun_out/pk_base.txt 2>&1; echo base_rc=$?
timeout 300 ncu --kernel-name regex:oz_pack --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/create_once.py 10000 2>/dev/null | grep -i "oz_pack" | tail -3 > gpurun_out/pk_ncu_base.csv
cp /tmp/libgls_new.so paper_1210_7325_b200/libgls.so
timeout 300 ncu --kernel-name regex:oz_pack --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/create_once.py 10000 2>/dev/null | grep -i "oz_pack" | tail -3 > gpurun_out/pk_ncu_new.csv
diff gpurun_out/pk_new.txt gpurun_out/pk_base.txt && echo DIGESTS_EQUAL
cat gpurun_out/pk_new.txt
echo base; cut -d, -f5,13- gpurun_out/pk_ncu_base.csv; echo new; cut -d, -f5,13- gpurun_out/pk_ncu_new.csv
