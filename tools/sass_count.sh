cnt () 
{ 
    awk -v a="/\\\\*$2\\\\*/" -v b="/\\\\*$3\\\\*/" '$0 ~ a {f=1} f{print} $0 ~ b {f=0}' $1 | grep -oP '^\s+/\*[0-9a-f]+\*/\s+\K[@!P0-9 ]*[A-Z][A-Z0-9_.]+' | sed 's/^@!*P[0-9T] //' | awk '{print $1}' | sed 's/\..*//' | sort | uniq -c | sort -rn | awk '{s+=$1; printf "%s:%s ",$2,$1} END {print " total",s}'
}
