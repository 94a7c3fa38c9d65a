"""`python -m paper_2505_21070_b200 <subcommand> ...`: the blockpipe CLI
(run / verify / plan / analyze / noise-demo) over the B200 engine."""
import sys

from .operator import cli_main


def main() -> int:
    code, out, err = cli_main(sys.argv[1:])
    sys.stdout.write(out)
    sys.stderr.write(err)
    return code


if __name__ == "__main__":
    sys.exit(main())
