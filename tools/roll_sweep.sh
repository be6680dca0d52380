#!/bin/bash
# dev: time the C2 step with alternative builds of the library (lib/libR*.so)
cp paper_2408_06213_b200/lib/libbatchrand_b200.so /tmp/orig.so
for f in paper_2408_06213_b200/lib/libR*.so; do
  cp $f paper_2408_06213_b200/lib/libbatchrand_b200.so; touch -d "+1 hour" paper_2408_06213_b200/lib/libbatchrand_b200.so
  echo "$f $(python tools/roll_overhead.py 2>&1 | head -2 | tr '\n' ' ')"
done
cp /tmp/orig.so paper_2408_06213_b200/lib/libbatchrand_b200.so; touch -d "+1 hour" paper_2408_06213_b200/lib/libbatchrand_b200.so
echo "orig $(python tools/roll_overhead.py 2>&1 | head -2 | tr '\n' ' ')"
