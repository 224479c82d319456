"""Datalog source language: scanner, recursive-descent parser, AST.

The accepted language is the reference's Souffle-like subset (reference:
pkg/README.md "Source language" EBNF; pkg/src/flatlog/parser.py:1-355):

    .decl Name(a:symbol, b:symbol)      relation declaration (arity >= 1)
    .input Name / .output Name          I/O marks
    .split label { A(..), B(..) } -> Helper(v1, .., vk)
    [label:] Head(t, ..) [:- [!]Body(t, ..), ..] .

Terms: bare identifiers are variables, `_` is a fresh anonymous variable,
quoted strings and decimal digit runs are constants (numbers stay strings,
as in the reference). `//` starts a comment.

Validation performed here (same error wording as the reference so callers
matching on messages keep working): range restriction of head variables,
safety of negated atoms, ground facts, declared relations and arities.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

from .faults import ProgramError

VAR = "var"
CONST = "const"

ANON_PREFIX = "_#"  # anonymous variables are renamed to _#<n>
_anon_counter = itertools.count(1)


@dataclass(frozen=True)
class Term:
    kind: str
    value: str

    def is_var(self) -> bool:
        return self.kind == VAR

    @property
    def anonymous(self) -> bool:
        return self.kind == VAR and self.value.startswith(ANON_PREFIX)


@dataclass(frozen=True)
class Atom:
    relation: str
    args: tuple
    negated: bool = False

    @property
    def arity(self) -> int:
        return len(self.args)

    def variables(self) -> list:
        return [t.value for t in self.args if t.kind == VAR]

    def __str__(self):
        parts = [t.value if t.kind == VAR else f'"{t.value}"' for t in self.args]
        return ("!" if self.negated else "") + f"{self.relation}({', '.join(parts)})"


@dataclass(frozen=True)
class Rule:
    head: Atom
    body: tuple
    index: int
    label: str | None = None

    @property
    def rule_id(self) -> str:
        return self.label if self.label else f"r{self.index}"

    def __str__(self):
        if not self.body:
            return f"{self.head}."
        return f"{self.head} :- " + ", ".join(str(a) for a in self.body) + "."


@dataclass(frozen=True)
class SplitDirective:
    rule_label: str
    subset: tuple
    helper_name: str
    helper_vars: tuple
    line: int


@dataclass
class Program:
    declarations: dict = field(default_factory=dict)  # relation -> arity
    inputs: list = field(default_factory=list)
    outputs: list = field(default_factory=list)
    rules: list = field(default_factory=list)
    facts: dict = field(default_factory=dict)  # relation -> [constant tuples]
    splits: list = field(default_factory=list)

    def arity(self, name: str) -> int:
        return self.declarations[name]


# --------------------------------------------------------------------------
# scanner

_PUNCT = set("().,:{}!")
_IDENT_START = set("abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ_")
_IDENT_BODY = _IDENT_START | set("0123456789?")


@dataclass(frozen=True)
class Token:
    kind: str  # ident | string | number | punct | implies | arrow | eof
    text: str
    line: int
    col: int


def scan(source: str) -> list:
    out = []
    i, n = 0, len(source)
    line, line_start = 1, 0
    while i < n:
        ch = source[i]
        col = i - line_start + 1
        if ch == "\n":
            line += 1
            i += 1
            line_start = i
            continue
        if ch.isspace():
            i += 1
            continue
        if source.startswith("//", i):
            j = source.find("\n", i)
            i = n if j < 0 else j
            continue
        if ch == '"':
            j = i + 1
            while j < n and source[j] not in '"\n':
                j += 1
            if j >= n or source[j] != '"':
                raise ProgramError(f"unexpected character {ch!r}", line, col)
            out.append(Token("string", source[i : j + 1], line, col))
            i = j + 1
            continue
        if ch.isdigit() and ch.isascii():
            j = i
            while j < n and source[j].isdigit() and source[j].isascii():
                j += 1
            out.append(Token("number", source[i:j], line, col))
            i = j
            continue
        if ch in _IDENT_START:
            j = i + 1
            while j < n and source[j] in _IDENT_BODY:
                j += 1
            out.append(Token("ident", source[i:j], line, col))
            i = j
            continue
        if source.startswith(":-", i):
            out.append(Token("implies", ":-", line, col))
            i += 2
            continue
        if source.startswith("->", i):
            out.append(Token("arrow", "->", line, col))
            i += 2
            continue
        if ch in _PUNCT:
            out.append(Token("punct", ch, line, col))
            i += 1
            continue
        raise ProgramError(f"unexpected character {ch!r}", line, col)
    out.append(Token("eof", "", line, i - line_start + 1))
    return out


# --------------------------------------------------------------------------
# parser


class _Reader:
    def __init__(self, source: str):
        self.toks = scan(source)
        self.at = 0
        self.prog = Program()

    # token helpers
    def look(self, k: int = 0) -> Token:
        return self.toks[min(self.at + k, len(self.toks) - 1)]

    def take(self) -> Token:
        tok = self.toks[self.at]
        if tok.kind != "eof":
            self.at += 1
        return tok

    def want(self, kind: str, text: str | None = None) -> Token:
        tok = self.take()
        if tok.kind != kind or (text is not None and tok.text != text):
            raise ProgramError(f"expected {(text or kind)!r}, found {tok.text!r}", tok.line, tok.col)
        return tok

    def is_punct(self, text: str, k: int = 0) -> bool:
        tok = self.look(k)
        return tok.kind == "punct" and tok.text == text

    def comma_list(self, item):
        items = [item()]
        while self.is_punct(","):
            self.take()
            items.append(item())
        return items

    # grammar
    def program(self) -> Program:
        while self.look().kind != "eof":
            if self.is_punct("."):
                self.directive()
            else:
                self.clause()
        self.check_references()
        return self.prog

    def directive(self):
        dot = self.want("punct", ".")
        word = self.want("ident")
        if word.text == "decl":
            self.declaration()
        elif word.text == "input":
            self.prog.inputs.append(self.want("ident").text)
        elif word.text == "output":
            self.prog.outputs.append(self.want("ident").text)
        elif word.text == "split":
            self.split(dot)
        else:
            raise ProgramError(f"unknown directive .{word.text}", word.line, word.col)

    def declaration(self):
        name = self.want("ident")
        if name.text in self.prog.declarations:
            raise ProgramError(f"relation {name.text} declared twice", name.line, name.col)
        self.want("punct", "(")

        def attribute():
            self.want("ident")
            if self.is_punct(":"):
                self.take()
                self.want("ident")  # the attribute type; everything is a symbol
            return 1

        arity = len(self.comma_list(attribute))
        self.want("punct", ")")
        self.prog.declarations[name.text] = arity

    def split(self, dot: Token):
        label = self.want("ident").text
        self.want("punct", "{")
        subset = self.comma_list(self.atom)
        self.want("punct", "}")
        self.want("arrow")
        helper = self.want("ident").text
        self.want("punct", "(")
        columns = self.comma_list(lambda: self.want("ident").text)
        self.want("punct", ")")
        for a in subset:
            if a.negated:
                raise ProgramError(f"cannot split on negated atom {a}", dot.line, dot.col)
        self.prog.splits.append(SplitDirective(label, tuple(subset), helper, tuple(columns), dot.line))

    def clause(self):
        label = None
        if self.look().kind == "ident" and self.is_punct(":", 1):
            label = self.take().text
            self.take()
        start = self.look()
        head = self.atom()
        if head.negated:
            raise ProgramError("rule head cannot be negated", start.line, start.col)
        body = []
        if self.look().kind == "implies":
            self.take()
            body = self.comma_list(self.atom)
        self.want("punct", ".")
        if not body:
            if any(t.kind == VAR for t in head.args):
                raise ProgramError(f"fact {head} contains variables", start.line, start.col)
            self.prog.facts.setdefault(head.relation, []).append(tuple(t.value for t in head.args))
            return
        _check_safety(head, body, start)
        self.prog.rules.append(Rule(head, tuple(body), len(self.prog.rules), label))

    def atom(self) -> Atom:
        negated = False
        if self.is_punct("!"):
            self.take()
            negated = True
        name = self.want("ident")
        self.want("punct", "(")
        args = self.comma_list(self.term)
        self.want("punct", ")")
        return Atom(name.text, tuple(args), negated)

    def term(self) -> Term:
        tok = self.take()
        if tok.kind == "ident":
            if tok.text == "_":
                return Term(VAR, f"{ANON_PREFIX}{next(_anon_counter)}")
            return Term(VAR, tok.text)
        if tok.kind == "string":
            return Term(CONST, tok.text[1:-1])
        if tok.kind == "number":
            return Term(CONST, tok.text)
        raise ProgramError(f"expected a term, found {tok.text!r}", tok.line, tok.col)

    def check_references(self):
        decls = self.prog.declarations

        def arity_ok(name, arity, where):
            want = decls.get(name)
            if want is None:
                raise ProgramError(f"relation {name} used in {where} but never declared")
            if want != arity:
                raise ProgramError(
                    f"{where}: relation {name} declared with arity {want}, used with {arity}"
                )

        for rule in self.prog.rules:
            where = f"rule {rule.rule_id}"
            for a in (rule.head, *rule.body):
                arity_ok(a.relation, a.arity, where)
        for name, rows in self.prog.facts.items():
            for row in rows:
                arity_ok(name, len(row), "fact")
        for name in (*self.prog.inputs, *self.prog.outputs):
            if name not in decls:
                raise ProgramError(f"relation {name} marked input/output but never declared")


def _check_safety(head: Atom, body: list, where: Token):
    bound = {v for a in body if not a.negated for v in a.variables()}
    for v in head.variables():
        if v not in bound:
            raise ProgramError(
                f"head variable {v} is not bound by a positive body atom", where.line, where.col
            )
    for a in body:
        if not a.negated:
            continue
        for v in a.variables():
            if not v.startswith(ANON_PREFIX) and v not in bound:
                raise ProgramError(
                    f"variable {v} of negated atom {a} is not bound by a positive atom",
                    where.line,
                    where.col,
                )


def parse(source: str) -> Program:
    """Parse Datalog text into a Program; raises ProgramError on bad input."""
    return _Reader(source).program()
