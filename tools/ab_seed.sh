bash tools/ab_variant.sh sr2 | grep -v "^base" | sed 's/^var/sr2/'
bash tools/ab_variant.sh sr8
