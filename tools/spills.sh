# usage: spills.sh <sass-with-line-info> <mangled-kernel-substring>: source lines of LDL/STL in one kernel
start=$(grep -n "^\.text\..*$2" "$1" | head -1 | cut -d: -f1)
awk -v s="$start" 'NR>=s && /^\.text\./ && NR>s {exit} NR>=s' "$1" | awk '/\/\/## File/{loc=$0} /LDL|STL/{print loc}' | sed 's/.*csrc\/\(.*\)", line \([0-9]*\).*/\1:\2/' | sort | uniq -c | sort -rn | head -${3:-25}
