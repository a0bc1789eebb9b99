cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/normal_variants.py 10 0x2c0a 0xc0a > gpurun_out/nv.txt 2>&1
for V in 10 0x2c0a; do
SFB_NORMAL_VARIANT=$V timeout 600 ncu --set full --clock-control none --import-source on -k regex:fill_normal_fast -s 1 -c 1 -f -o gpurun_out/prof_normal_$V python tools/prof_driver.py normal > gpurun_out/ncu_normal_$V.txt 2>&1
done
cat gpurun_out/nv.txt
